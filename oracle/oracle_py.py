"""TEST INFRASTRUCTURE ONLY: ctypes access to the CPU checkers.

* ``libgd_oracle.so`` -- the plain-C restatement (gd_oracle.c).
* ``_ref/libgdref.so`` -- the reference headers compiled from
  /root/reference (ref_harness.cpp); present only where it was built.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` legs import this module.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from pathlib import Path

import numpy as np

from paper_1901_06363_b200.native import (DockResult, LigandBatch, Knobs, gd_knobs,
                                          gd_ligand_batch, gd_result)

HERE = Path(__file__).resolve().parent
ORACLE_LIB = HERE / "libgd_oracle.so"
REF_LIB = HERE / "_ref" / "libgdref.so"
REF_INC = Path("/root/reference/proj/include")

_i32p = C.POINTER(C.c_int32)
_i64p = C.POINTER(C.c_longlong)
_f64p = C.POINTER(C.c_double)
_u8p = C.POINTER(C.c_uint8)


def _p(a, t):
    return a.ctypes.data_as(t) if a is not None else None


def build(ref: bool = True) -> None:
    """make the oracle (and, where /root/reference exists, oracle/_ref)."""
    targets = ["all"] + (["ref"] if ref and REF_INC.exists() else [])
    subprocess.run(["make", "-s", "-C", str(HERE), *targets], check=True)


_oracle = None
_ref = None


def oracle() -> C.CDLL:
    global _oracle
    if _oracle is None:
        if not ORACLE_LIB.exists():
            build(ref=False)
        h = C.CDLL(str(ORACLE_LIB))
        h.gdo_overlap_score.restype = C.c_double
        h.gdo_overlap_score.argtypes = [_f64p, C.c_int, _f64p, C.c_int]
        h.gdo_optimal_tile_size.argtypes = [C.c_int]
        h.gdo_dock_batch.argtypes = [C.POINTER(gd_ligand_batch), _f64p, C.c_int,
                                     C.POINTER(gd_knobs), C.c_int, C.POINTER(gd_result)]
        h.gdo_match_probes_shape.argtypes = [C.c_int, _f64p, _f64p, C.c_int, _i32p, _u8p, _f64p,
                                             C.c_int, C.POINTER(gd_knobs), _f64p, _f64p, _i64p,
                                             _i64p]
        h.gdo_rotate_fragment.argtypes = [C.c_int, _f64p, _f64p, C.c_int, _i32p, _u8p, _f64p,
                                          C.c_int, C.c_double, _f64p, C.POINTER(C.c_int)]
        h.gdo_orientations.argtypes = [C.c_int, C.POINTER(_i32p), C.POINTER(_f64p)]
        h.gdo_pocket_centre.argtypes = [_f64p, C.c_int, _f64p]
        h.gdo_free.argtypes = [C.c_void_p]
        h.gdo_rotation_profiles.argtypes = [C.c_int, _f64p, _f64p, C.c_int, _i32p, _u8p, _f64p,
                                            C.c_int, _f64p, _u8p, _f64p, C.c_int,
                                            C.POINTER(C.c_int)]
        _oracle = h
    return _oracle


def have_ref() -> bool:
    return REF_LIB.exists()


def ref() -> C.CDLL:
    global _ref
    if _ref is None:
        if not REF_LIB.exists():
            if not REF_INC.exists():
                raise RuntimeError("oracle/_ref was not built and /root/reference is absent")
            build(ref=True)
        h = C.CDLL(str(REF_LIB))
        h.gdref_last_error.restype = C.c_char_p
        h.gdref_overlap_score.restype = C.c_double
        h.gdref_overlap_score.argtypes = [_f64p, C.c_int, _f64p, C.c_int, C.c_int]
        h.gdref_optimal_tile_size.argtypes = [C.c_int]
        h.gdref_match_probes_shape.argtypes = [C.c_int, _f64p, _f64p, C.c_int, _i32p, _u8p,
                                               _f64p, C.c_int, C.POINTER(gd_knobs), C.c_int,
                                               _f64p, _f64p, _i64p, _i64p]
        h.gdref_rotate_fragment.argtypes = [C.c_int, _f64p, _f64p, C.c_int, _i32p, _u8p, _f64p,
                                            C.c_int, C.c_double, _f64p, C.POINTER(C.c_int)]
        h.gdref_generate_synthetic.argtypes = [C.c_int, C.c_uint64, C.c_int, C.c_int, C.c_int,
                                               C.c_int, C.c_int, C.c_double, C.POINTER(C.c_int),
                                               C.POINTER(C.c_int), _f64p, _i32p, _f64p, _f64p,
                                               _i32p, _i32p, _u8p]
        h.gdref_dock_batch.argtypes = [C.POINTER(gd_ligand_batch), _f64p, C.c_int,
                                       C.POINTER(gd_knobs), C.c_int, C.c_int,
                                       C.POINTER(gd_result)]
        h.gdref_rotation_profiles.restype = C.c_longlong
        h.gdref_rotation_profiles.argtypes = [C.POINTER(gd_ligand_batch), _f64p, C.c_int, C.c_int,
                                              C.c_int, _f64p, _u8p, _f64p, _i32p, _i32p,
                                              C.c_longlong]
        h.gdref_detect_peaks.argtypes = [_f64p, _u8p, _f64p, C.POINTER(C.c_int),
                                         C.POINTER(C.c_int), _i32p, _i32p, _f64p]
        h.gdref_tile_hits.argtypes = [_i32p, C.c_int, _i32p, C.c_int, _f64p, _f64p]
        h.gdref_ligand_graph.argtypes = [C.c_int, _f64p, _f64p, C.c_int, _i32p, _u8p, _i32p, _u8p]
        _ref = h
    return _ref


def threads() -> int:
    return len(os.sched_getaffinity(0))


# ---------------------------------------------------------------------------
def dock_batch(batch: LigandBatch, pocket: np.ndarray, knobs: Knobs, nthreads: int = 1,
               keep_poses: bool = True, impl: str = "oracle", use_index: bool = True) -> DockResult:
    """E1-E8 on the CPU: impl 'oracle' (C restatement) or 'ref' (reference headers)."""
    pk = np.ascontiguousarray(pocket, dtype=np.float64)
    res = DockResult.empty(batch.n_ligands, knobs.slots, int(batch.atom_offsets[-1]), keep_poses)
    b, k, r = batch.c_struct(), knobs.c_struct(), res.c_struct()
    if impl == "oracle":
        oracle().gdo_dock_batch(C.byref(b), _p(pk, _f64p), len(pk), C.byref(k), nthreads, C.byref(r))
    else:
        ref().gdref_dock_batch(C.byref(b), _p(pk, _f64p), len(pk), C.byref(k), nthreads,
                               int(use_index), C.byref(r))
    return res


def overlap_score(xyz: np.ndarray, pocket: np.ndarray, impl: str = "oracle",
                  use_index: bool = False) -> float:
    x = np.ascontiguousarray(xyz, dtype=np.float64)
    pk = np.ascontiguousarray(pocket, dtype=np.float64)
    if impl == "oracle":
        return oracle().gdo_overlap_score(_p(x, _f64p), len(x), _p(pk, _f64p), len(pk))
    return ref().gdref_overlap_score(_p(x, _f64p), len(x), _p(pk, _f64p), len(pk), int(use_index))


def match_probes_shape(xyz, radii, bonds, rot, pocket, knobs: Knobs, impl: str = "oracle",
                       use_index: bool = False):
    """(score, evaluations, feasibility_checks, final_pose) or raises RuntimeError."""
    x = np.ascontiguousarray(xyz, dtype=np.float64)
    r = np.ascontiguousarray(radii, dtype=np.float64)
    b = np.ascontiguousarray(bonds, dtype=np.int32)
    ro = np.ascontiguousarray(rot, dtype=np.uint8)
    pk = np.ascontiguousarray(pocket, dtype=np.float64)
    out = np.zeros_like(x)
    sc = C.c_double()
    ev = C.c_longlong()
    ck = C.c_longlong()
    k = knobs.c_struct()
    if impl == "oracle":
        rc = oracle().gdo_match_probes_shape(len(x), _p(x, _f64p), _p(r, _f64p), len(b),
                                             _p(b, _i32p), _p(ro, _u8p), _p(pk, _f64p), len(pk),
                                             C.byref(k), _p(out, _f64p), C.byref(sc),
                                             C.byref(ev), C.byref(ck))
        if rc:
            raise RuntimeError(f"oracle error {rc}")
    else:
        rc = ref().gdref_match_probes_shape(len(x), _p(x, _f64p), _p(r, _f64p), len(b),
                                            _p(b, _i32p), _p(ro, _u8p), _p(pk, _f64p), len(pk),
                                            C.byref(k), int(use_index), _p(out, _f64p),
                                            C.byref(sc), C.byref(ev), C.byref(ck))
        if rc:
            raise RuntimeError(ref().gdref_last_error().decode())
    return sc.value, ev.value, ck.value, out


def optimize_fragment(xyz, radii, bonds, rot, pocket, f: int, step: int, refined: bool = False,
                      pose=None, entry_score: float = -1.0):
    """optimize_fragment_flat / _refined on fragment f: (best_angle, best_score, evals,
    checks, committed pose)."""
    h = oracle()
    h.gdo_optimize_fragment.argtypes = [C.c_int, _f64p, _f64p, C.c_int, _i32p, _u8p, _f64p,
                                        C.c_int, _f64p, C.c_int, C.c_int, C.c_int, C.c_double,
                                        _f64p, C.POINTER(C.c_int), _f64p, _i64p, _i64p]
    x = np.ascontiguousarray(xyz, dtype=np.float64)
    r = np.ascontiguousarray(radii, dtype=np.float64)
    b = np.ascontiguousarray(bonds, dtype=np.int32).reshape(-1, 2)
    ro = np.ascontiguousarray(rot, dtype=np.uint8)
    pk = np.ascontiguousarray(pocket, dtype=np.float64)
    p = x if pose is None else np.ascontiguousarray(pose, dtype=np.float64)
    out = np.zeros_like(x)
    ang, sc, ev, ck = C.c_int(), C.c_double(), C.c_longlong(), C.c_longlong()
    rc = h.gdo_optimize_fragment(len(x), _p(x, _f64p), _p(r, _f64p), len(b), _p(b, _i32p),
                                 _p(ro, _u8p), _p(pk, _f64p), len(pk), _p(p, _f64p), f,
                                 int(refined), step, entry_score, _p(out, _f64p), C.byref(ang),
                                 C.byref(sc), C.byref(ev), C.byref(ck))
    if rc:
        raise RuntimeError(f"oracle error {rc}")
    return ang.value, sc.value, ev.value, ck.value, out


def ref_optimize_fragment(xyz, radii, bonds, rot, pocket, f: int, step: int,
                          refined: bool = False, pose=None, entry_score=None):
    """The reference's optimize_fragment_flat / _refined (kernel.hpp:125-198)
    on fragment f: (best_angle, best_score, evals, checks, committed pose)."""
    h = ref()
    h.gdref_optimize_fragment.argtypes = [C.c_int, _f64p, _f64p, C.c_int, _i32p, _u8p, _f64p,
                                          C.c_int, _f64p, C.c_int, C.c_int, C.c_int, C.c_int,
                                          C.c_double, _f64p, C.POINTER(C.c_int), _f64p, _i64p,
                                          _i64p]
    x = np.ascontiguousarray(xyz, dtype=np.float64)
    r = np.ascontiguousarray(radii, dtype=np.float64)
    b = np.ascontiguousarray(bonds, dtype=np.int32).reshape(-1, 2)
    ro = np.ascontiguousarray(rot, dtype=np.uint8)
    pk = np.ascontiguousarray(pocket, dtype=np.float64)
    p = x if pose is None else np.ascontiguousarray(pose, dtype=np.float64)
    out = np.zeros_like(x)
    ang, sc, ev, ck = C.c_int(), C.c_double(), C.c_longlong(), C.c_longlong()
    rc = h.gdref_optimize_fragment(len(x), _p(x, _f64p), _p(r, _f64p), len(b), _p(b, _i32p),
                                   _p(ro, _u8p), _p(pk, _f64p), len(pk), _p(p, _f64p), f,
                                   int(refined), step, int(entry_score is not None),
                                   0.0 if entry_score is None else float(entry_score),
                                   _p(out, _f64p), C.byref(ang), C.byref(sc), C.byref(ev),
                                   C.byref(ck))
    if rc:
        raise RuntimeError(h.gdref_last_error().decode())
    return ang.value, sc.value, ev.value, ck.value, out


def rotate_fragment(xyz, radii, bonds, rot, pose, f: int, angle: float, impl: str = "oracle"):
    """(rotated pose, feasible) for fragment f (rotamer f//2; left if f even)."""
    x = np.ascontiguousarray(xyz, dtype=np.float64)
    r = np.ascontiguousarray(radii, dtype=np.float64)
    b = np.ascontiguousarray(bonds, dtype=np.int32)
    ro = np.ascontiguousarray(rot, dtype=np.uint8)
    p = np.ascontiguousarray(pose, dtype=np.float64)
    out = np.zeros_like(x)
    feas = C.c_int()
    fn = oracle().gdo_rotate_fragment if impl == "oracle" else ref().gdref_rotate_fragment
    rc = fn(len(x), _p(x, _f64p), _p(r, _f64p), len(b), _p(b, _i32p), _p(ro, _u8p), _p(p, _f64p),
            f, angle, _p(out, _f64p), C.byref(feas))
    if rc:
        msg = ref().gdref_last_error().decode() if impl != "oracle" else f"oracle error {rc}"
        raise RuntimeError(msg)
    return out, bool(feas.value)


def rotation_profiles(batch: LigandBatch, pocket: np.ndarray, impl: str = "oracle",
                      nthreads: int = 1):
    """rotation_profile (analysis.hpp:37-56) of every fragment of every ligand
    from its batch pose, laid out like gd_rotation_profiles: returns
    (scores [F,360], valid [F,360] bool, relative_size [F], frag_offsets
    [L+1], status [L]).  impl 'oracle' = C restatement (brute force), 'ref'
    = the reference's own rotation_profile with its PocketIndex."""
    pk = np.ascontiguousarray(pocket, dtype=np.float64)
    L = batch.n_ligands
    cap = max(1, 2 * int(batch.rotatable.sum()))
    scores = np.zeros((cap, 360), np.float64)
    valid = np.zeros((cap, 360), np.uint8)
    rel = np.zeros(cap, np.float64)
    offs = np.zeros(L + 1, np.int32)
    status = np.zeros(max(L, 1), np.int32)
    if impl == "oracle":
        nfrag = C.c_int()
        for l in range(L):
            xyz, radii, bonds, rot = batch.ligand(l)
            o = int(offs[l])
            rc = oracle().gdo_rotation_profiles(
                len(xyz), _p(xyz, _f64p), _p(radii, _f64p), len(bonds), _p(bonds, _i32p),
                _p(rot, _u8p), _p(pk, _f64p), len(pk), _p(scores[o:], _f64p), _p(valid[o:], _u8p),
                _p(rel[o:], _f64p), cap - o, C.byref(nfrag))
            if rc < 0:
                raise RuntimeError("rotation_profiles: capacity")
            status[l] = rc
            offs[l + 1] = o + nfrag.value
    else:
        b = batch.c_struct()
        n = ref().gdref_rotation_profiles(C.byref(b), _p(pk, _f64p), len(pk), 1, nthreads,
                                          _p(scores, _f64p), _p(valid, _u8p), _p(rel, _f64p),
                                          _p(offs, _i32p), _p(status, _i32p), cap)
        if n < 0:
            raise RuntimeError("rotation_profiles: capacity")
    F = int(offs[-1])
    return scores[:F], valid[:F].astype(bool), rel[:F], offs, status[:L]


def ref_detect_peaks(scores, valid):
    """The reference detect_peaks (analysis.hpp:61-126): (delta, best_peak_width,
    [(start, width, height_ratio), ...]) or None when it throws."""
    s = np.ascontiguousarray(scores, dtype=np.float64)
    v = np.ascontiguousarray(valid, dtype=np.uint8)
    d, bw, npk = C.c_double(), C.c_int(), C.c_int()
    st = np.zeros(360, np.int32)
    wd = np.zeros(360, np.int32)
    ht = np.zeros(360, np.float64)
    if ref().gdref_detect_peaks(_p(s, _f64p), _p(v, _u8p), C.byref(d), C.byref(bw), C.byref(npk),
                                _p(st, _i32p), _p(wd, _i32p), _p(ht, _f64p)):
        return None
    k = npk.value
    return d.value, bw.value, [(int(st[i]), int(wd[i]), float(ht[i])) for i in range(k)]


def ref_tile_hits(best_widths, tiles):
    """The reference tile_hit_probability (analysis.hpp:133-147)."""
    bw = np.ascontiguousarray(best_widths, dtype=np.int32)
    t = np.ascontiguousarray(tiles, dtype=np.int32)
    prob = np.zeros(len(t))
    ev = np.zeros(len(t))
    if ref().gdref_tile_hits(_p(bw, _i32p), len(bw), _p(t, _i32p), len(t), _p(prob, _f64p),
                             _p(ev, _f64p)):
        raise RuntimeError(ref().gdref_last_error().decode())
    return prob, ev


def ref_ligand_graph(xyz, radii, bonds, rot):
    """The reference's find_rotamers + grow_fragments: (bond indices, membership)
    or None when the Ligand ctor throws."""
    x = np.ascontiguousarray(xyz, dtype=np.float64)
    r = np.ascontiguousarray(radii, dtype=np.float64)
    b = np.ascontiguousarray(bonds, dtype=np.int32)
    ro = np.ascontiguousarray(rot, dtype=np.uint8)
    n, nb = len(x), len(b)
    rb = np.zeros(max(nb, 1), np.int32)
    mem = np.zeros((max(2 * nb, 1), max(n, 1)), np.uint8)
    k = ref().gdref_ligand_graph(n, _p(x, _f64p), _p(r, _f64p), nb, _p(b, _i32p), _p(ro, _u8p),
                                 _p(rb, _i32p), _p(mem, _u8p))
    if k < 0:
        return None
    return rb[:k].copy(), mem[:2 * k, :n].astype(bool)


def orientations(step: int):
    idx = _i32p()
    R = _f64p()
    n = oracle().gdo_orientations(step, C.byref(idx), C.byref(R))
    i = np.ctypeslib.as_array(idx, shape=(n,)).copy()
    m = np.ctypeslib.as_array(R, shape=(n * 9,)).copy().reshape(n, 3, 3)
    oracle().gdo_free(C.cast(idx, C.c_void_p))
    oracle().gdo_free(C.cast(R, C.c_void_p))
    return i, m


def pocket_centre(pocket) -> np.ndarray:
    pk = np.ascontiguousarray(pocket, dtype=np.float64)
    c = np.zeros(3)
    oracle().gdo_pocket_centre(_p(pk, _f64p), len(pk), _p(c, _f64p))
    return c


def ref_generate_synthetic(count, seed, atom_lo=6, atom_hi=14, rot_lo=2, rot_hi=4,
                           pocket_points=60, pocket_radius=8.0):
    """The reference's own generator (synthetic.hpp:71-188): (pocket, LigandBatch)."""
    h = ref()
    ta, tb = C.c_int(), C.c_int()
    args = [count, seed, atom_lo, atom_hi, rot_lo, rot_hi, pocket_points, pocket_radius]
    if h.gdref_generate_synthetic(*args, C.byref(ta), C.byref(tb), None, None, None, None, None,
                                  None, None):
        raise RuntimeError(h.gdref_last_error().decode())
    pocket = np.zeros((pocket_points, 3))
    ao = np.zeros(count + 1, np.int32)
    xyz = np.zeros((ta.value, 3))
    radii = np.zeros(ta.value)
    bo = np.zeros(count + 1, np.int32)
    bonds = np.zeros((tb.value, 2), np.int32)
    rot = np.zeros(tb.value, np.uint8)
    h.gdref_generate_synthetic(*args, C.byref(ta), C.byref(tb), _p(pocket, _f64p), _p(ao, _i32p),
                               _p(xyz, _f64p), _p(radii, _f64p), _p(bo, _i32p), _p(bonds, _i32p),
                               _p(rot, _u8p))
    return pocket, LigandBatch(ao, xyz, radii, bo, bonds, rot)
