"""Summarise an A/B log: variant, ligands/s, ms/step, per-kernel ms."""
import json
import sys

v = None
for line in open(sys.argv[1]):
    if line.startswith("variant"):
        v = line.strip()
    elif line.startswith("{"):
        d = json.loads(line)
        print(v, round(d["value"]), round(d["ms_per_step"], 3),
              {k: round(x, 3) for k, x in d.get("kernel_ms", {}).items()})
