"""Shared test utilities: result comparison and small hand-built ligands."""
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


class Lig:
    """A hand-built ligand: positions, radii, bonds (a, b, rotatable)."""

    def __init__(self, positions, bonds, radius=1.0):
        self.xyz = np.array(positions, dtype=np.float64).reshape(-1, 3)
        self.radii = np.full(len(self.xyz), float(radius)) if np.isscalar(radius) \
            else np.array(radius, dtype=np.float64)
        self.bonds = np.array([[a, b] for a, b, _ in bonds], dtype=np.int32).reshape(-1, 2)
        self.rot = np.array([int(r) for _, _, r in bonds], dtype=np.uint8)

    @property
    def args(self):
        return self.xyz, self.radii, self.bonds, self.rot

    def batch(self):
        from paper_1901_06363_b200 import LigandBatch
        return LigandBatch([0, len(self.xyz)], self.xyz, self.radii, [0, len(self.bonds)],
                           self.bonds, self.rot)


def chain(positions, radius=1.0, rotatable=None):
    """chain_ligand (reference tests/support/test_helpers.hpp:14-32)."""
    n = len(positions)
    rot = rotatable if rotatable is not None else [True] * (n - 1)
    return Lig(positions, [(i - 1, i, rot[i - 1]) for i in range(1, n)], radius)


def peak_rig():
    """PeakRig (reference test_kernel.cpp:19-31): profile peaks at 90 degrees."""
    lig = Lig([[0, 0, 0], [0, 0, 1], [1, 0, 1]], [(0, 1, True), (1, 2, False)])
    pocket = np.array([[0, 0, 0], [0, 0, 1.2], [0, -1, 1]], dtype=np.float64)
    return lig, pocket


def bump_probe(separation, radius):
    """bump_probe_ligand (reference test_geometry.cpp:176-187)."""
    pos = [[1.5 * i, 0.0, 0.0] for i in range(6)]
    pos[5] = [0.0, separation, 0.0]
    pos[4] = [1.5, separation, 0.0]
    pos[3] = [3.0, separation, 0.0]
    return Lig(pos, [(i, i + 1, i == 2) for i in range(5)], radius)
