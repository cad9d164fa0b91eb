"""Rotation-profile analysis (reference analysis.hpp:17-217) over the C-ABI.

The profiles come from the GPU (``gd_rotation_profiles``), peak extraction
and the tile-hit model from the native host code (``gd_detect_peaks``,
``gd_tile_hit_probability``); this module only arranges their results into
the reference's row types.  Fragment f of a ligand is rotamer f // 2, left
if f is even (kernel.hpp:221-227).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from .native import (GD_ERR_INVALID, GD_OK, Docker, GeoDockError, Knobs, LigandBatch, Profiles,
                     _p, lib)


class gd_peak(C.Structure):
    _fields_ = [("start_angle", C.c_int32), ("width", C.c_int32), ("height_ratio", C.c_double)]


@dataclass
class Peak:
    start_angle: int
    width: int
    height_ratio: float


@dataclass
class PeakStats:
    delta_overlap: float = 0.0
    peaks: list = field(default_factory=list)
    best_peak_width: int = 0


@dataclass
class TileHit:
    tile_size: int
    probability: float
    eval_count: float


@dataclass
class FragmentProfileRow:
    ligand_id: str
    rotamer_index: int
    side: str  # "left" | "right"
    relative_size: float
    delta_overlap: float
    delta_normalized: float
    peak_count: int
    best_peak_width: int


@dataclass
class PeakRow:
    ligand_id: str
    rotamer_index: int
    side: str
    start_angle: int
    width: int
    height_ratio: float


@dataclass
class LigandAnalysis:
    score: float          # PoseResult.score of the dock
    evaluations: int
    feasibility_checks: int
    final_pose: np.ndarray
    fragments: list = field(default_factory=list)
    peaks: list = field(default_factory=list)
    stats: list = field(default_factory=list)


def detect_peaks(scores: np.ndarray, valid: np.ndarray) -> PeakStats:
    """detect_peaks (analysis.hpp:61-126); raises GeoDockError when no angle is valid."""
    s = np.ascontiguousarray(scores, dtype=np.float64)
    v = np.ascontiguousarray(valid, dtype=np.uint8)
    delta, best, npk = C.c_double(), C.c_int32(), C.c_int32()
    buf = (gd_peak * 360)()
    rc = lib().gd_detect_peaks(_p(s, C.POINTER(C.c_double)), _p(v, C.POINTER(C.c_uint8)),
                               C.byref(delta), C.byref(best), C.cast(buf, C.c_void_p),
                               C.byref(npk))
    if rc != GD_OK:
        raise GeoDockError(rc, "detect_peaks: no feasible rotation")
    return PeakStats(delta.value, [Peak(buf[k].start_angle, buf[k].width, buf[k].height_ratio)
                                   for k in range(npk.value)], best.value)


def tile_hit_probability(dataset: list, tile_sizes: list) -> list:
    """tile_hit_probability (analysis.hpp:133-147) over PeakStats (or best widths)."""
    widths = np.array([d.best_peak_width if isinstance(d, PeakStats) else int(d) for d in dataset],
                      dtype=np.int32)
    tiles = np.ascontiguousarray(tile_sizes, dtype=np.int32)
    prob = np.zeros(len(tiles))
    ev = np.zeros(len(tiles))
    rc = lib().gd_tile_hit_probability(_p(widths, C.POINTER(C.c_int32)), len(widths),
                                       _p(tiles, C.POINTER(C.c_int32)), len(tiles),
                                       _p(prob, C.POINTER(C.c_double)),
                                       _p(ev, C.POINTER(C.c_double)))
    if rc != GD_OK:
        raise GeoDockError(GD_ERR_INVALID, "tile_hit_probability: empty dataset")
    return [TileHit(int(t), float(p), float(e)) for t, p, e in zip(tiles, prob, ev)]


def analyze_ligands(docker: Docker, batch: LigandBatch, knobs: Knobs,
                    ids: list | None = None) -> list:
    """analyze_ligand (analysis.hpp:177-215) for a whole batch on the GPU:
    match_probes_shape from each ligand's given pose, then the rotation
    profile of every fragment from the final committed pose.  Fragments
    with no feasible rotation are skipped, as in the reference.  Ligands
    that fail validation or hit a degenerate axis yield None."""
    k = Knobs(**{**knobs.__dict__, "rigid_step": 0, "top_k": 1})
    res = docker.dock(batch, k, keep_poses=True)
    L = batch.n_ligands
    final = LigandBatch(batch.atom_offsets, res.final_pose.reshape(-1, 3), batch.radii,
                        batch.bond_offsets, batch.bonds, batch.rotatable)
    prof: Profiles = docker.rotation_profiles(final)
    out = []
    for l in range(L):
        if res.status[l] != 0 or prof.status[l] != 0:
            out.append(None)
            continue
        lid = ids[l] if ids is not None else str(l)
        a0, a1 = batch.atom_offsets[l], batch.atom_offsets[l + 1]
        la = LigandAnalysis(float(res.final_score[l, 0]), int(res.evaluations[l, 0]),
                            int(res.feasibility_checks[l, 0]), final.xyz[a0:a1].copy())
        for f in range(int(prof.frag_offsets[l]), int(prof.frag_offsets[l + 1])):
            try:
                st = detect_peaks(prof.scores[f], prof.valid[f])
            except GeoDockError:
                continue  # no feasible rotation for this fragment
            fl = f - int(prof.frag_offsets[l])
            side = "left" if fl % 2 == 0 else "right"
            la.fragments.append(FragmentProfileRow(
                lid, fl // 2, side, float(prof.relative_size[f]), st.delta_overlap,
                st.delta_overlap / la.score if la.score > 0.0 else 0.0, len(st.peaks),
                st.best_peak_width))
            la.peaks.extend(PeakRow(lid, fl // 2, side, p.start_angle, p.width, p.height_ratio)
                            for p in st.peaks)
            la.stats.append(st)
        out.append(la)
    return out
