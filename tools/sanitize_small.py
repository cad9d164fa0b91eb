"""Small GPU workload for compute-sanitizer runs: config 0, 32 config-1
ligands, two large ligands (multi-word masks, narrowed CTAs), the refined
search, a K > 32 rigid top-K, and rotation profiles.
    compute-sanitizer --tool memcheck python tools/sanitize_small.py"""
import os
import sys

sys.path.insert(0, os.getcwd())
from paper_1901_06363_b200 import Docker, Knobs, synth_ligands, workloads as W  # noqa: E402

d = Docker(0)
w0 = W.config(0)
d.set_pocket(w0.pocket())
d.dock(w0.ligands(), w0.knobs, keep_poses=True)
w1 = W.config(1)
p1 = w1.pocket()
d.set_pocket(p1)
b = w1.ligands(range(32), p1.mean(axis=0))
d.dock(b, w1.knobs, keep_poses=True)
d.dock(b, Knobs(20, 45, 0.25, 2, True, 45, 40))
big = synth_ligands(777, [0, 1], n_lo=150, n_hi=256, r_cap=12, centre=p1.mean(axis=0))
d.dock(big, Knobs(90, 90, 0.0, 1, False, 90, 3), keep_poses=True)
prof = d.rotation_profiles(b)
# GPU preprocessing corner cases and the top-1 pose output.
from paper_1901_06363_b200 import LigandBatch  # noqa: E402
bad = b.subset(range(6))
bad.radii[bad.atom_offsets[2]] = -1.0
bad.bonds[bad.bond_offsets[4]] = [0, 0]
d.dock(bad, w1.knobs, top_pose=True)
d.dock(b, w1.knobs, top_pose=True)
d.upload(b)
d.dock_resident(w1.knobs, top_pose=True)
print("sanitize run ok", len(prof.scores))
