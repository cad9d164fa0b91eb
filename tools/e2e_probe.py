import sys, time, json
sys.path.insert(0, '.')
import numpy as np, torch
from paper_1901_06363_b200 import Docker, workloads as W
w = W.config(1); pocket = w.pocket(); batch = w.ligands(range(10000), pocket.mean(axis=0))
d = Docker(0); d.set_pocket(pocket)
for i in range(4):
    t0 = time.perf_counter(); d.dock(batch, w.knobs); dt = time.perf_counter() - t0
    print(json.dumps({"wall_ms": dt * 1e3, **{k: v for k, v in d.timing().items() if 'ms' in k}}))
