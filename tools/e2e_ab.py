"""e2e A/B of gd_dock_batch settings on config 1, as bench.py's e2e leg
measures it (host buffers reused, L2 flushed, top-1 poses fetched).

    python tools/e2e_ab.py "GD_E2E_HEAD=256" "GD_E2E_HEAD=512 GD_E2E_GROWTH=2" ...
Each setting runs in its own process (the knobs are read once per process);
prints the median of 7 calls per setting, and per-setting device time.
"""
import json
import os
import statistics
import subprocess
import sys

CHILD = r"""
import sys, time, json, statistics
sys.path.insert(0, '.')
import torch
from paper_1901_06363_b200 import Docker, workloads as W
w = W.config(1); pocket = w.pocket(); batch = w.ligands(range(10000), pocket.mean(axis=0))
d = Docker(0); d.set_pocket(pocket)
flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
out = d.dock(batch, w.knobs, top_pose=True)
ts = []
for i in range(7):
    flush.zero_(); torch.cuda.synchronize()
    t0 = time.perf_counter(); d.dock(batch, w.knobs, out=out, top_pose=True); ts.append(time.perf_counter() - t0)
t = d.timing()
print(json.dumps({"e2e_ms": 1e3 * statistics.median(ts), "best_ms": 1e3 * min(ts),
                  "pack_ms": t["host_pack_ms"], "post_ms": t["host_post_ms"]}))
"""


def main():
    for cfg in sys.argv[1:] or [""]:
        env = dict(os.environ)
        for kv in cfg.split():
            k, v = kv.split("=", 1)
            env[k] = v
        r = subprocess.run([sys.executable, "-c", CHILD], env=env, capture_output=True, text=True)
        line = r.stdout.strip().splitlines()[-1] if r.stdout.strip() else r.stderr[-400:]
        print(json.dumps({"setting": cfg, "result": line}), flush=True)


if __name__ == "__main__":
    main()
