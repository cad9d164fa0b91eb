"""BASELINE config 4: the accuracy / time-to-solution trade-off on the GPU.

Knob grid: rigid step {10,15,20,30,45}, fragment step {10,20,30,60}
(lp = max(45, step)), restarts {1,2,3}, K {10,30,100} over config-3-style
pockets (semi-axes U(5,12) A, 1 A lattice, roughness).  For every point:
device time-to-solution per ligand-pocket dock, and the Eq. 4 degradation
(reference overlap_degradation, screening.hpp:190-193: 1 - top1%mean /
top1%mean_finest, in %) of each ligand's top-pose score against the finest
point (10, 10, 3, 100).

    python tools/knob_sweep.py --ligands 500 --pockets 4 [--full] > profiles/r1_knob_sweep.json
"""
from __future__ import annotations

import argparse
import itertools
import json
import math
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

from paper_1901_06363_b200 import Docker, Knobs, workloads as W  # noqa: E402


def top1pct_mean(scores: np.ndarray) -> float:
    """top1pct_mean_score (reference screening.hpp:78-89)."""
    k = max(1, math.ceil(0.01 * len(scores)))
    return float(np.sort(scores)[::-1][:k].mean())


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ligands", type=int, default=500)
    ap.add_argument("--pockets", type=int, default=4)
    ap.add_argument("--full", action="store_true", help="all 180 grid points (else a 36-point subset)")
    a = ap.parse_args()
    w = W.config(4)
    rigid = [10, 15, 20, 30, 45]
    frag = [10, 20, 30, 60]
    reps = [1, 2, 3]
    ks = [10, 30, 100]
    grid = list(itertools.product(rigid, frag, reps, ks))
    if not a.full:
        grid = [g for g in grid if g[2] in (1, 3) and g[3] in (10, 100) and g[1] != 20] + [(10, 10, 3, 100)]
        grid = sorted(set(grid))
    finest = (10, 10, 3, 100)
    d = Docker(0)
    pockets = [W.pocket_of(w, p) for p in range(a.pockets)]
    batches = [w.ligands(range(a.ligands), pk.mean(axis=0)) for pk in pockets]
    results = {}
    for g in grid:
        knobs = Knobs.baseline(*g)
        tops, ms, poses = [], 0.0, 0
        for pk, b in zip(pockets, batches):
            d.set_pocket(pk)
            d.upload(b)
            d.dock_resident(knobs)  # warm
            t0 = time.perf_counter()
            d.dock_resident(knobs)
            t = d.timing()
            ms += t["rigid_ms"] + t["flex_ms"]
            from paper_1901_06363_b200.native import DockResult
            r = d.download(DockResult.empty(b.n_ligands, knobs.slots, int(b.atom_offsets[-1]), False))
            tops.append(r.final_score[:, 0])
            poses += int(r.poses_scored.sum())
        results[g] = {"device_ms": ms, "top": np.concatenate(tops), "poses": poses}
    ref = top1pct_mean(results[finest]["top"])
    out = []
    for g, r in sorted(results.items()):
        docks = a.ligands * a.pockets
        out.append({
            "rigid_step": g[0], "fragment_step": g[1], "restarts": g[2], "top_k": g[3],
            "device_ms": r["device_ms"], "docks_per_s": docks / (r["device_ms"] / 1e3),
            "poses_scored": r["poses"],
            "degradation_pct": (1.0 - top1pct_mean(r["top"]) / ref) * 100.0,
            "mean_top_pose_rel_delta": float(np.mean((results[finest]["top"] - r["top"]) / results[finest]["top"])),
        })
    print(json.dumps({"workload": f"config 4 style: {a.ligands} ligands x {a.pockets} pockets",
                      "finest": finest, "points": out}, indent=1))


if __name__ == "__main__":
    main()
