"""Where the analysis e2e time goes: gd_upload vs gd_rotation_profiles, with
pageable vs pinned host output buffers.  python tools/profiles_e2e_probe.py"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
from paper_1901_06363_b200 import Docker, workloads as W  # noqa: E402
from paper_1901_06363_b200.native import ProfileBuffers  # noqa: E402

w = W.config(1)
pocket = w.pocket()
batch = w.ligands(range(2000), pocket.mean(axis=0))
d = Docker(0)
d.set_pocket(pocket)
out = ProfileBuffers.for_batch(batch)
pin = ProfileBuffers.for_batch(batch)
for name in ("scores", "valid", "rel"):
    a = getattr(pin, name)
    t = torch.empty(a.shape, dtype=torch.from_numpy(a[:0]).dtype, pin_memory=True)
    setattr(pin, name, t.numpy())
for label, buf in (("pageable", out), ("pinned", pin)):
    for _ in range(3):
        d.rotation_profiles(batch, out=buf)
    up, pr = [], []
    for _ in range(5):
        t0 = time.perf_counter()
        d.upload(batch)
        t1 = time.perf_counter()
        d.rotation_profiles(out=buf)
        t2 = time.perf_counter()
        up.append(t1 - t0)
        pr.append(t2 - t1)
    print(f"{label:9s} upload {1e3 * np.mean(up):6.2f} ms  profiles+D2H {1e3 * np.mean(pr):6.2f} ms  "
          f"kernel {d.timing()['flex_ms']:.2f} ms")
