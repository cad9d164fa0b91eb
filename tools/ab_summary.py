"""Summarise gpurun_out/ab_*.log: per variant, ms per step and kernel times."""
import json
import sys

cur = None
for line in open(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/ab_src.log"):
    if line.startswith("variant"):
        cur = line.strip()
    elif line.startswith("{"):
        d = json.loads(line)
        k = d.get("kernel_ms", {})
        print(f"{cur:60s} {d['ms_per_step']:8.3f} ms  " + "  ".join(f"{n.split('_')[0]} {v:.3f}" for n, v in k.items()))
