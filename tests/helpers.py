"""Shared test utilities: result comparison and small datasets."""
from __future__ import annotations

import numpy as np

FIELDS = ["orientation", "seed_rank", "rigid_score", "final_score", "evaluations",
          "feasibility_checks", "k_eff", "poses_scored", "status"]


def assert_same_result(got, want, poses: bool = True, ctx: str = ""):
    """Bit-exact equality of two DockResults (indices, ordering, fp64 scores, counters)."""
    for f in FIELDS:
        a, b = getattr(got, f), getattr(want, f)
        if not np.array_equal(a, b):
            bad = np.argwhere(a != b)
            raise AssertionError(f"{ctx}{f} differs at {bad[:5].tolist()}: "
                                 f"got {a[tuple(bad[0])]!r} want {b[tuple(bad[0])]!r}")
    if poses and want.final_pose is not None and got.final_pose is not None:
        if not np.array_equal(got.final_pose, want.final_pose):
            d = np.abs(got.final_pose - want.final_pose)
            raise AssertionError(f"{ctx}final_pose differs: max |d| {d.max():.3e}")


def bits(x: np.ndarray) -> np.ndarray:
    return np.ascontiguousarray(x, dtype=np.float64).view(np.uint64)
