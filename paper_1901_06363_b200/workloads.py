"""BASELINE.json configurations as seeded synthetic workloads.

The paper's 113K-ligand library and PDB pockets are not available
(reference PAPER.md:552-554), so seeded synthetic inputs with BASELINE's
shapes stand in for them (DESIGN.md §5 records the choices):

* Pockets are lattice ellipsoids.  Configs 0/1 state 2,000 / 4,000 points "on
  a 1 A lattice", which is inconsistent (a 1 A lattice gives 983 / 1,989);
  we honour the point counts with a 0.795 A lattice (1,983 / 3,991 points).
  Configs 3/4 use a true 1 A lattice and the roughness mask.
* Ligands: random-walk trees (csrc/synth.cpp), n ~ U{20..60} (32 in config
  0), rotatable bonds ~ U{0..min(12, n/4)} (6 in config 0), radii
  U(1.2, 1.9) A, centroid on the pocket centre.
* Knobs: BASELINE's (rigid step, fragment step, restarts, K) mapped onto
  KnobConfig{step, max(45, step), 0.0, restarts, false}.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .native import Knobs, LigandBatch, synth_ligands, synth_pocket

SPACING_STATED_COUNT = 0.795  # A; gives the stated 2,000 / 4,000 points
BASE_SEED = 0x1901063600000000


@dataclass
class Workload:
    name: str
    n_ligands: int
    pocket_axes: tuple
    spacing: float
    knobs: Knobs
    fixed_n: int = 0
    fixed_r: int = -1
    rough_max: float = 0.0
    seed: int = BASE_SEED
    notes: str = ""
    pockets: list = field(default_factory=list)

    def pocket(self) -> np.ndarray:
        a, b, c = self.pocket_axes
        return synth_pocket(a, b, c, self.spacing, self.rough_max, self.seed)

    def ligands(self, ids=None, centre=None) -> LigandBatch:
        if ids is None:
            ids = range(self.n_ligands)
        if centre is None:
            centre = self.pocket().mean(axis=0)
        return synth_ligands(self.seed, ids, 20, 60, self.fixed_n, 12, self.fixed_r, centre)


def config(i: int) -> Workload:
    if i == 0:
        return Workload("c0: 1 ligand (n=32, R=6) x 1 pocket 8x6x5 A, rigid 30, frag 30, 1 restart, K=30",
                        1, (8.0, 6.0, 5.0), SPACING_STATED_COUNT, Knobs.baseline(30, 30, 1, 30),
                        fixed_n=32, fixed_r=6, seed=BASE_SEED + 0)
    if i == 1:
        return Workload("c1: 10,000 ligands x 1 pocket 10x8x6 A, rigid 30, frag 30, 1 restart, K=30",
                        10_000, (10.0, 8.0, 6.0), SPACING_STATED_COUNT,
                        Knobs.baseline(30, 30, 1, 30), seed=BASE_SEED + 1)
    if i == 2:
        return Workload("c2: 2,000 ligands x 1 pocket 10x8x6 A, rigid 10, frag 10, 3 restarts, K=100",
                        2_000, (10.0, 8.0, 6.0), SPACING_STATED_COUNT,
                        Knobs.baseline(10, 10, 3, 100), seed=BASE_SEED + 2)
    if i in (3, 4):
        rng = np.random.default_rng(BASE_SEED + i)
        n_pockets = 16 if i == 3 else 4
        axes = [tuple(rng.uniform(5.0, 12.0, 3)) for _ in range(n_pockets)]
        w = Workload(f"c{i}: {'100,000' if i == 3 else '20,000'} ligands x {n_pockets} pockets "
                     "(semi-axes U(5,12) A, 1 A lattice, roughness U(0,20%))",
                     100_000 if i == 3 else 20_000, axes[0], 1.0, Knobs.baseline(30, 30, 1, 30),
                     rough_max=0.2, seed=BASE_SEED + i)
        w.pockets = axes
        return w
    raise ValueError(i)


def pocket_of(w: Workload, p: int) -> np.ndarray:
    """Pocket p of a multi-pocket workload (configs 3/4)."""
    a, b, c = w.pockets[p] if w.pockets else w.pocket_axes
    return synth_pocket(a, b, c, w.spacing, w.rough_max, w.seed + 1000 + p)


def synth_pocket_unrough(w: Workload, p: int) -> np.ndarray:
    """Pocket p before its roughness mask (to report the removed fraction)."""
    a, b, c = w.pockets[p] if w.pockets else w.pocket_axes
    return synth_pocket(a, b, c, w.spacing, 0.0, w.seed + 1000 + p)
