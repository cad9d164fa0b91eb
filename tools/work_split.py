"""Executed work of both kernels on a config (GPU): pairs per query etc.
python tools/work_split.py [config]"""
import os
import sys

sys.path.insert(0, os.getcwd())
from paper_1901_06363_b200 import Docker, Knobs, workloads as W  # noqa: E402
from paper_1901_06363_b200.native import GD_FLAG_COUNT_WORK  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 1
w = W.config(cfg)
pocket = w.pocket()
d = Docker(0)
d.set_pocket(pocket)
d.upload(w.ligands(range(min(w.n_ligands, 10000)), pocket.mean(axis=0)))
d.dock_resident(Knobs(**{**w.knobs.__dict__, "flags": GD_FLAG_COUNT_WORK}))
for k, v in d.work_counters().items():
    q = max(1, v["queries"])
    print(k, v, f"pairs/query {v['pairs'] / q:.3f}")
