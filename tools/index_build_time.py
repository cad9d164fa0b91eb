"""Wall time of gd_set_pocket (voxel index build) on config 1 and the
largest config-3 pockets.  python tools/index_build_time.py"""
import os
import sys
import time

sys.path.insert(0, os.getcwd())
from paper_1901_06363_b200 import Docker, workloads as W  # noqa: E402

d = Docker(0)
cases = [("c1", W.config(1).pocket())]
w3 = W.config(3)
pockets = [W.pocket_of(w3, i) for i in range(16)]
pockets.sort(key=len)
cases += [(f"c3 P={len(pockets[0])}", pockets[0]), (f"c3 P={len(pockets[-1])}", pockets[-1])]
for name, pk in cases:
    d.set_pocket(pk)  # warm
    t0 = time.perf_counter()
    for _ in range(3):
        d.set_pocket(pk)
    dt = (time.perf_counter() - t0) / 3
    info = d.pocket_info()
    print(f"{name:14s} points={len(pk):5d} build={dt * 1e3:8.2f} ms  dims={info['dims'].tolist()} "
          f"h={info['voxel']:.3f} candidates={info['n_candidates']}")
