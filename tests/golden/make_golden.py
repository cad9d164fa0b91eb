"""Regenerate tests/golden/*.npz from the reference itself.

Run in the build container (needs /root/reference): the reference headers
are compiled from their own sources into oracle/_ref/libgdref.so
(oracle/Makefile) and every output below comes from reference calls:
geodock::generate_synthetic, geodock::match_probes_shape,
geodock::overlap_score, geodock::optimal_tile_size, geodock::rotate_fragment /
check_bumps, and the E1-E8 batch path of oracle/ref_harness.cpp (reference
overlap_score + match_probes_shape per seed).

    python tests/golden/make_golden.py
"""
from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ROOT = HERE.parent.parent
sys.path.insert(0, str(ROOT))

from oracle import oracle_py as O  # noqa: E402
from paper_1901_06363_b200 import Knobs, workloads as W  # noqa: E402

# Knob settings the reference's own tests use (test_kernel.cpp, test_screening.cpp).
REF_KNOBS = [
    (1, 45, 0.0, 1, False),
    (2, 90, 0.3, 2, True),
    (5, 90, 0.3, 1, False),
    (3, 45, 0.2, 1, True),
    (10, 90, 0.5, 1, False),
    (1, 90, 1.0, 1, False),
]
# (count, seed, atom_lo, atom_hi, rot_lo, rot_hi, points): the reference
# tests' small_dataset calls (test_kernel.cpp:206, :223, :242, :253,
# test_geometry.cpp:217, :237).
REF_DATASETS = [
    (10, 321, 6, 14, 2, 4, 60),
    (5, 555, 6, 14, 2, 4, 60),
    (12, 4242, 6, 14, 2, 4, 60),
    (6, 9001, 6, 14, 2, 4, 60),
    (10, 2024, 6, 14, 2, 4, 60),
    (12, 31, 6, 14, 2, 4, 120),
]


def batch_arrays(prefix, b):
    return {f"{prefix}atom_offsets": b.atom_offsets, f"{prefix}xyz": b.xyz,
            f"{prefix}radii": b.radii, f"{prefix}bond_offsets": b.bond_offsets,
            f"{prefix}bonds": b.bonds, f"{prefix}rotatable": b.rotatable}


def result_arrays(prefix, r):
    out = {}
    for f in ("orientation", "seed_rank", "rigid_score", "final_score", "evaluations",
              "feasibility_checks", "k_eff", "poses_scored", "status", "final_pose"):
        out[prefix + f] = getattr(r, f)
    return out


def make_reference_kernel():
    """match_probes_shape on the reference generator's datasets, per knob set."""
    out = {"knobs": np.array([[k[0], k[1], k[2], k[3], int(k[4])] for k in REF_KNOBS])}
    for d, (count, seed, alo, ahi, rlo, rhi, pts) in enumerate(REF_DATASETS):
        pocket, b = O.ref_generate_synthetic(count, seed, alo, ahi, rlo, rhi, pts, 8.0)
        out[f"d{d}_pocket"] = pocket
        out.update(batch_arrays(f"d{d}_", b))
        for ki, k in enumerate(REF_KNOBS):
            knobs = Knobs(*k)
            scores, ev, ck, poses = [], [], [], []
            for l in range(b.n_ligands):
                x, r, bd, ro = b.ligand(l)
                s, e, c, p = O.match_probes_shape(x, r, bd, ro, pocket, knobs, impl="ref")
                scores.append(s)
                ev.append(e)
                ck.append(c)
                poses.append(p)
            out[f"d{d}_k{ki}_score"] = np.array(scores)
            out[f"d{d}_k{ki}_evals"] = np.array(ev)
            out[f"d{d}_k{ki}_checks"] = np.array(ck)
            out[f"d{d}_k{ki}_pose"] = np.concatenate(poses)
    out["tile_sizes"] = np.array([O.ref().gdref_optimal_tile_size(s) for s in range(1, 361)])
    np.savez_compressed(HERE / "reference_kernel.npz", **out)


def make_baseline_configs():
    """E1-E8 (reference calls) on BASELINE-shaped inputs: c0 whole, c1 and c2 subsets."""
    out = {}
    cases = [("c0", W.config(0), None), ("c1", W.config(1), list(range(6))),
             ("c2", W.config(2), [5])]
    for name, w, ids in cases:
        pocket = w.pocket()
        b = w.ligands(ids, pocket.mean(axis=0))
        r = O.dock_batch(b, pocket, w.knobs, nthreads=O.threads(), impl="ref", use_index=True)
        out[f"{name}_pocket"] = pocket
        out[f"{name}_knobs"] = np.array([w.knobs.high_precision_step, w.knobs.low_precision_step,
                                         w.knobs.threshold, w.knobs.repetitions,
                                         int(w.knobs.enable_refinement), w.knobs.rigid_step,
                                         w.knobs.top_k])
        out.update(batch_arrays(f"{name}_", b))
        out.update(result_arrays(f"{name}_", r))
    np.savez_compressed(HERE / "baseline_configs.npz", **out)


if __name__ == "__main__":
    O.build(ref=True)
    make_reference_kernel()
    make_baseline_configs()
    for f in sorted(HERE.glob("*.npz")):
        print(f.name, f.stat().st_size)
