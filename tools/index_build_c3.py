"""gd_set_pocket wall time, index footprint and record format per config-3
pocket, first and second build.
python tools/index_build_c3.py"""
import os
import sys
import time

sys.path.insert(0, os.getcwd())
from paper_1901_06363_b200 import Docker, workloads as W  # noqa: E402

d = Docker(0)
d.set_pocket(W.config(1).pocket())  # context + module warm-up
w3 = W.config(3)
for i in range(16):
    pk = W.pocket_of(w3, i)
    t0 = time.perf_counter()
    d.set_pocket(pk)
    t1 = time.perf_counter()
    d.set_pocket(pk)
    t2 = time.perf_counter()
    info = d.pocket_info()
    print(f"pocket {i:2d} P={len(pk):5d} first={1e3 * (t1 - t0):7.1f} ms second={1e3 * (t2 - t1):7.1f} ms "
          f"dims={info['dims'].tolist()} h={info['voxel']:.3f} cand={info['n_candidates']} "
          f"index={info['index_bytes'] / 1e6:.1f} MB {info['format']}")
