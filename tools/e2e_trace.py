"""Per-chunk e2e timeline of gd_dock_batch on config 1 (GD_E2E_TRACE=1):
host prep interval and GPU start/end of every chunk, relative to the call.
Run: GD_E2E_TRACE=1 python tools/e2e_trace.py"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1901_06363_b200 import Docker, workloads as W  # noqa: E402

w = W.config(1)
pocket = w.pocket()
batch = w.ligands(range(10000), pocket.mean(axis=0))
d = Docker(0)
d.set_pocket(pocket)
out = None
for i in range(4):
    t0 = time.perf_counter()
    out = d.dock(batch, w.knobs, out=out)
    print(f"--- call {i}: wall {1e3 * (time.perf_counter() - t0):.3f} ms", file=sys.stderr, flush=True)
