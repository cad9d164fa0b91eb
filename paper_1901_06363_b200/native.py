"""ctypes binding of the C-ABI in include/geodock_b200.h.

This is plumbing for the tests and the benchmark; the product is the
native library.  Loading fails loudly if ``libgeodock_b200.so`` is missing:
there is no Python or CPU fallback for any hot-path call.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from pathlib import Path

import numpy as np

LIB_PATH = Path(__file__).resolve().parent / "libgeodock_b200.so"

GD_OK = 0
GD_ERR_INVALID = 1
GD_ERR_CUDA = 2
GD_ERR_DEGENERATE = 3
GD_ERR_NO_POCKET = 4
GD_LIG_OK = 0
GD_LIG_INVALID = 1
GD_LIG_DEGENERATE = 3
GD_FLAG_BRUTE_FORCE = 1
GD_FLAG_KEEP_POSES = 2
GD_FLAG_COUNT_WORK = 4
GD_FLAG_TOP_POSE = 16
WORK_FIELDS = ["pairs", "rotated", "bump_pairs", "queries", "sum_terms", "evaluations", "xform"]

_i32p = C.POINTER(C.c_int32)
_i64p = C.POINTER(C.c_int64)
_f64p = C.POINTER(C.c_double)
_u8p = C.POINTER(C.c_uint8)


class gd_ligand_batch(C.Structure):
    _fields_ = [("n_ligands", C.c_int32), ("atom_offsets", _i32p), ("xyz", _f64p),
                ("radii", _f64p), ("bond_offsets", _i32p), ("bonds", _i32p),
                ("bond_rotatable", _u8p)]


class gd_knobs(C.Structure):
    _fields_ = [("high_precision_step", C.c_int32), ("low_precision_step", C.c_int32),
                ("threshold", C.c_double), ("repetitions", C.c_int32),
                ("enable_refinement", C.c_int32), ("rigid_step", C.c_int32),
                ("top_k", C.c_int32), ("flags", C.c_uint32)]


class gd_result(C.Structure):
    _fields_ = [("orientation", _i32p), ("seed_rank", _i32p), ("rigid_score", _f64p),
                ("final_score", _f64p), ("evaluations", _i64p),
                ("feasibility_checks", _i64p), ("final_pose", _f64p), ("k_eff", _i32p),
                ("poses_scored", _i64p), ("status", _i32p), ("top_pose", _f64p)]


class gd_device_result(C.Structure):
    _fields_ = [("orientation", C.c_void_p), ("seed_rank", C.c_void_p),
                ("final_score", C.c_void_p), ("evaluations", C.c_void_p),
                ("n_ligands", C.c_int32), ("top_k", C.c_int32),
                ("rigid_score", C.c_void_p), ("feasibility_checks", C.c_void_p),
                ("k_eff", C.c_void_p), ("poses_scored", C.c_void_p), ("status", C.c_void_p)]


class gd_fragment_set(C.Structure):
    _fields_ = [("membership", _u8p), ("axis_atom", _i32p), ("anchor_atom", _i32p)]


class _CudaArray:
    """__cuda_array_interface__ view of a device buffer owned by the library
    (lets torch wrap it without a copy, e.g. for an NCCL all-gather)."""

    def __init__(self, ptr: int, shape, typestr: str):
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": typestr,
                                         "data": (ptr, False), "version": 3, "strides": None}


class gd_timing(C.Structure):
    _fields_ = [("upload_ms", C.c_float), ("rigid_ms", C.c_float), ("flex_ms", C.c_float),
                ("download_ms", C.c_float), ("total_ms", C.c_float),
                ("rigid_atom_queries", C.c_int64), ("flex_atom_queries", C.c_int64),
                ("launches", C.c_int64), ("h2d_bytes", C.c_int64), ("d2h_bytes", C.c_int64),
                ("host_prep_ms", C.c_float), ("host_pack_ms", C.c_float),
                ("host_post_ms", C.c_float)]


class gd_index_level(C.Structure):
    _fields_ = [("dims", C.c_int32 * 3), ("voxel", C.c_double), ("candidates", C.c_int64),
                ("record_bytes", C.c_int64), ("list_bytes", C.c_int64)]


class gd_multi_stats(C.Structure):
    _fields_ = [("ligands", C.c_int64), ("chunks", C.c_int64), ("busy_ms", C.c_float)]


# Every symbol include/geodock_b200.h declares, with its ctypes signature.
SIGNATURES = {
    "gd_create": (C.c_int, [C.c_int, C.POINTER(C.c_void_p)]),
    "gd_destroy": (C.c_int, [C.c_void_p]),
    "gd_last_error": (C.c_char_p, [C.c_void_p]),
    "gd_set_stream": (C.c_int, [C.c_void_p, C.c_void_p]),
    "gd_version": (C.c_char_p, []),
    "gd_set_pocket": (C.c_int, [C.c_void_p, _f64p, C.c_int32]),
    "gd_pocket_info": (C.c_int, [C.c_void_p, _f64p, _i32p, _f64p, _i64p, _i32p]),
    "gd_dock_batch": (C.c_int, [C.c_void_p, C.POINTER(gd_ligand_batch), C.POINTER(gd_knobs),
                                C.POINTER(gd_result)]),
    "gd_upload": (C.c_int, [C.c_void_p, C.POINTER(gd_ligand_batch)]),
    "gd_dock_resident": (C.c_int, [C.c_void_p, C.POINTER(gd_knobs)]),
    "gd_download": (C.c_int, [C.c_void_p, C.POINTER(gd_result)]),
    "gd_last_timing": (C.c_int, [C.c_void_p, C.POINTER(gd_timing)]),
    "gd_work_counters": (C.c_int, [C.c_void_p, C.POINTER(C.c_uint64)]),
    "gd_phase_clocks": (C.c_int, [C.c_void_p, C.POINTER(C.c_uint64)]),
    "gd_ligand_graph": (C.c_int, [C.c_int32, C.POINTER(C.c_double), C.POINTER(C.c_double),
                                  C.c_int32, C.POINTER(C.c_int32), C.POINTER(C.c_uint8),
                                  C.POINTER(C.c_int32), C.POINTER(C.c_int32),
                                  C.POINTER(C.c_uint8), C.c_char_p, C.c_size_t]),
    "gd_cost_features": (None, [C.POINTER(C.c_double), C.POINTER(C.c_double)]),
    "gd_fit_cost_model": (C.c_int, [C.POINTER(C.c_double), C.POINTER(C.c_double), C.c_int32,
                                    C.POINTER(C.c_double), C.POINTER(C.c_double),
                                    C.POINTER(C.c_double), C.c_char_p, C.c_size_t]),
    "gd_l2_gather_peak": (C.c_int, [C.c_void_p, C.POINTER(C.c_double)]),
    "gd_detect_peaks": (C.c_int, [C.POINTER(C.c_double), C.POINTER(C.c_uint8),
                                  C.POINTER(C.c_double), C.POINTER(C.c_int32), C.c_void_p,
                                  C.POINTER(C.c_int32)]),
    "gd_tile_hit_probability": (C.c_int, [C.POINTER(C.c_int32), C.c_int64, C.POINTER(C.c_int32),
                                          C.c_int32, C.POINTER(C.c_double),
                                          C.POINTER(C.c_double)]),
    "gd_rotation_profiles": (C.c_int, [C.c_void_p, C.c_uint32, C.POINTER(C.c_double),
                                       C.POINTER(C.c_uint8),
                                       C.POINTER(C.c_double), C.POINTER(C.c_int32),
                                       C.POINTER(C.c_int32), C.c_int64]),
    "gd_device_results": (C.c_int, [C.c_void_p, C.POINTER(gd_device_result)]),
    "gd_l2_gather_rate": (C.c_int, [C.c_void_p, C.c_int32, C.POINTER(C.c_double)]),
    "gd_pocket_index_stats": (C.c_int, [C.c_void_p, C.POINTER(gd_index_level)]),
    "gd_pocket_index_format": (C.c_int, [C.c_void_p]),
    "gd_ligand_error": (C.c_int, [C.c_void_p, C.c_int32, C.c_char_p, C.c_size_t]),
    "gd_multi_create": (C.c_int, [_i32p, C.c_int32, C.POINTER(C.c_void_p)]),
    "gd_multi_destroy": (C.c_int, [C.c_void_p]),
    "gd_multi_last_error": (C.c_char_p, [C.c_void_p]),
    "gd_multi_size": (C.c_int32, [C.c_void_p]),
    "gd_multi_context": (C.c_void_p, [C.c_void_p, C.c_int32]),
    "gd_multi_set_pocket": (C.c_int, [C.c_void_p, _f64p, C.c_int32]),
    "gd_multi_dock_batch": (C.c_int, [C.c_void_p, C.POINTER(gd_ligand_batch), C.POINTER(gd_knobs),
                                      C.POINTER(gd_result)]),
    "gd_multi_last_stats": (C.c_int, [C.c_void_p, C.POINTER(gd_multi_stats), C.c_int32]),
    "gd_multi_ligand_error": (C.c_int, [C.c_void_p, C.c_int32, C.c_char_p, C.c_size_t]),
    "gd_optimize_fragment_batch": (C.c_int, [C.c_void_p, C.POINTER(gd_ligand_batch),
                                             C.POINTER(gd_fragment_set), C.c_int32, C.c_int32,
                                             _f64p, _i32p, _f64p, _i64p, _i64p, _f64p, _i32p]),
    "gd_rotate_fragment_batch": (C.c_int, [C.c_void_p, C.POINTER(gd_ligand_batch),
                                           C.POINTER(gd_fragment_set), _f64p, _f64p, _i32p]),
    "gd_check_bumps_batch": (C.c_int, [C.c_void_p, C.POINTER(gd_ligand_batch),
                                       C.POINTER(gd_fragment_set), _u8p, _i32p]),
    "gd_fp64_peak": (C.c_int, [C.c_void_p, C.POINTER(C.c_double)]),
    "gd_overlap_score_batch": (C.c_int, [C.c_void_p, _f64p, C.c_int32, C.c_int32, C.c_uint32,
                                         _f64p]),
    "gd_optimal_tile_size": (C.c_int32, [C.c_int32]),
    "gd_validate_knobs": (C.c_int, [C.POINTER(gd_knobs), C.c_char_p, C.c_size_t]),
    "gd_orientations": (C.c_int32, [C.c_int32, _i32p, _f64p, C.c_int32]),
    "gd_synth_pocket": (C.c_int32, [C.c_double, C.c_double, C.c_double, C.c_double,
                                    C.c_double, C.c_uint64, _f64p, C.c_int32]),
    "gd_synth_ligand_size": (C.c_int, [C.c_uint64, C.c_int64, C.c_int32, C.c_int32, C.c_int32,
                                       _i32p]),
    "gd_synth_ligand": (C.c_int, [C.c_uint64, C.c_int64, C.c_int32, C.c_int32, C.c_int32,
                                  C.c_int32, C.c_int32, _f64p, _f64p, _f64p, _i32p, _u8p]),
}

_lib = None


def lib() -> C.CDLL:
    """The loaded native library (raises if it was never built)."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise RuntimeError(
                f"{LIB_PATH} is missing: build it with `python -m paper_1901_06363_b200.build` "
                "(there is no CPU fallback)")
        h = C.CDLL(str(LIB_PATH))
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(h, name)
            fn.restype = res
            fn.argtypes = args
        _lib = h
    return _lib


def _p(a: np.ndarray, t):
    return a.ctypes.data_as(t) if a is not None else None


class GeoDockError(RuntimeError):
    """geodock::Error raised through the C-ABI (reference error.hpp:14-17)."""

    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code


# ---------------------------------------------------------------------------
# Inputs
# ---------------------------------------------------------------------------
@dataclass
class LigandBatch:
    """SoA ligand batch (gd_ligand_batch)."""
    atom_offsets: np.ndarray   # int32 [L+1]
    xyz: np.ndarray            # float64 [A, 3]
    radii: np.ndarray          # float64 [A]
    bond_offsets: np.ndarray   # int32 [L+1]
    bonds: np.ndarray          # int32 [B, 2]
    rotatable: np.ndarray      # uint8 [B]

    def __post_init__(self):
        self.atom_offsets = np.ascontiguousarray(self.atom_offsets, dtype=np.int32)
        self.xyz = np.ascontiguousarray(self.xyz, dtype=np.float64).reshape(-1, 3)
        self.radii = np.ascontiguousarray(self.radii, dtype=np.float64)
        self.bond_offsets = np.ascontiguousarray(self.bond_offsets, dtype=np.int32)
        self.bonds = np.ascontiguousarray(self.bonds, dtype=np.int32).reshape(-1, 2)
        self.rotatable = np.ascontiguousarray(self.rotatable, dtype=np.uint8)

    @property
    def n_ligands(self) -> int:
        return len(self.atom_offsets) - 1

    @property
    def sizes(self) -> np.ndarray:
        return np.diff(self.atom_offsets)

    def c_struct(self) -> gd_ligand_batch:
        return gd_ligand_batch(self.n_ligands, _p(self.atom_offsets, _i32p), _p(self.xyz, _f64p),
                               _p(self.radii, _f64p), _p(self.bond_offsets, _i32p),
                               _p(self.bonds, _i32p), _p(self.rotatable, _u8p))

    def ligand(self, l: int):
        a0, a1 = self.atom_offsets[l], self.atom_offsets[l + 1]
        b0, b1 = self.bond_offsets[l], self.bond_offsets[l + 1]
        return self.xyz[a0:a1], self.radii[a0:a1], self.bonds[b0:b1], self.rotatable[b0:b1]

    def subset(self, idx) -> "LigandBatch":
        parts = [self.ligand(int(l)) for l in idx]
        return LigandBatch.from_parts(parts)

    @staticmethod
    def from_parts(parts) -> "LigandBatch":
        ao = np.zeros(len(parts) + 1, np.int32)
        bo = np.zeros(len(parts) + 1, np.int32)
        for i, (x, _, b, _) in enumerate(parts):
            ao[i + 1] = ao[i] + len(x)
            bo[i + 1] = bo[i] + len(b)
        cat = lambda k, shape, dt: (np.concatenate([p[k] for p in parts]) if parts
                                    else np.zeros(shape, dt))
        return LigandBatch(ao, cat(0, (0, 3), np.float64), cat(1, (0,), np.float64), bo,
                           cat(2, (0, 2), np.int32), cat(3, (0,), np.uint8))


@dataclass
class Knobs:
    """KnobConfig (kernel.hpp:21-26) + the batch knobs."""
    high_precision_step: int = 1
    low_precision_step: int = 45
    threshold: float = 0.0
    repetitions: int = 3
    enable_refinement: bool = False
    rigid_step: int = 0
    top_k: int = 1
    flags: int = 0

    @staticmethod
    def baseline(rigid_step: int, frag_step: int, restarts: int, top_k: int) -> "Knobs":
        """BASELINE.json knob mapping: lp = max(45, step), threshold 0, no refinement."""
        return Knobs(frag_step, max(45, frag_step), 0.0, restarts, False, rigid_step, top_k)

    def c_struct(self) -> gd_knobs:
        return gd_knobs(self.high_precision_step, self.low_precision_step, self.threshold,
                        self.repetitions, int(bool(self.enable_refinement)), self.rigid_step,
                        self.top_k, self.flags)

    def validate(self) -> None:
        buf = C.create_string_buffer(256)
        k = self.c_struct()
        if lib().gd_validate_knobs(C.byref(k), buf, 256) != GD_OK:
            raise GeoDockError(GD_ERR_INVALID, buf.value.decode())

    @property
    def slots(self) -> int:
        return self.top_k if self.rigid_step > 0 else 1


class ProfileBuffers:
    """Host output buffers of gd_rotation_profiles, sized for a batch (2 x
    its rotatable bonds fragments) and reusable across calls."""

    def __init__(self, cap: int, n_ligands: int):
        self.scores = np.empty((cap, 360), np.float64)
        self.valid = np.empty((cap, 360), np.uint8)
        self.rel = np.empty(cap, np.float64)
        self.offs = np.empty(n_ligands + 1, np.int32)
        self.status = np.empty(max(n_ligands, 1), np.int32)

    @staticmethod
    def for_batch(batch: "LigandBatch") -> "ProfileBuffers":
        return ProfileBuffers(max(1, 2 * int(batch.rotatable.sum())), batch.n_ligands)

    def fits(self, batch: "LigandBatch") -> bool:
        return (len(self.rel) >= 2 * int(batch.rotatable.sum())
                and len(self.offs) >= batch.n_ligands + 1)


@dataclass
class Profiles:
    """Rotation profiles of a batch: fragment f of ligand l is row
    frag_offsets[l] + f (rotamer f // 2, left if f is even)."""
    scores: np.ndarray         # [F, 360] overlap score where valid, else 0
    valid: np.ndarray          # [F, 360] bool, check_bumps
    relative_size: np.ndarray  # [F]
    frag_offsets: np.ndarray   # [L+1]
    status: np.ndarray         # [L] GD_LIG_*


@dataclass
class DockResult:
    """gd_result as [L, K] numpy arrays (final order: score desc, seed rank asc)."""
    orientation: np.ndarray
    seed_rank: np.ndarray
    rigid_score: np.ndarray
    final_score: np.ndarray
    evaluations: np.ndarray
    feasibility_checks: np.ndarray
    k_eff: np.ndarray
    poses_scored: np.ndarray
    status: np.ndarray
    final_pose: np.ndarray | None = None  # flat [K*A*3] (see header for layout)
    top_pose: np.ndarray | None = None    # [A, 3]: each ligand's slot-0 pose at its atom offset

    @staticmethod
    def empty(L: int, K: int, total_atoms: int, poses: bool, top: bool = False) -> "DockResult":
        return DockResult(np.zeros((L, K), np.int32), np.zeros((L, K), np.int32),
                          np.zeros((L, K)), np.zeros((L, K)), np.zeros((L, K), np.int64),
                          np.zeros((L, K), np.int64), np.zeros(L, np.int32),
                          np.zeros(L, np.int64), np.zeros(L, np.int32),
                          np.zeros(K * total_atoms * 3) if poses else None,
                          np.zeros((total_atoms, 3)) if top else None)

    def fits(self, L: int, K: int, total_atoms: int, poses: bool, top: bool = False) -> bool:
        return (self.orientation.shape == (L, K)
                and (self.final_pose is not None) == poses
                and (not poses or len(self.final_pose) == K * total_atoms * 3)
                and (self.top_pose is not None) == top
                and (not top or self.top_pose.shape == (total_atoms, 3)))

    def c_struct(self) -> gd_result:
        return gd_result(_p(self.orientation, _i32p), _p(self.seed_rank, _i32p),
                         _p(self.rigid_score, _f64p), _p(self.final_score, _f64p),
                         _p(self.evaluations, _i64p), _p(self.feasibility_checks, _i64p),
                         _p(self.final_pose, _f64p), _p(self.k_eff, _i32p),
                         _p(self.poses_scored, _i64p), _p(self.status, _i32p),
                         _p(self.top_pose, _f64p))

    def pose(self, batch: LigandBatch, l: int, e: int) -> np.ndarray:
        K = self.orientation.shape[1]
        a0 = int(batch.atom_offsets[l])
        n = int(batch.atom_offsets[l + 1]) - a0
        off = 3 * (K * a0 + e * n)
        return self.final_pose[off:off + 3 * n].reshape(n, 3)


# ---------------------------------------------------------------------------
# Device context
# ---------------------------------------------------------------------------
class Docker:
    """One gd_ctx: a pocket staged on one GPU plus the resident batch."""

    def __init__(self, device: int = 0):
        self._lib = lib()
        h = C.c_void_p()
        rc = self._lib.gd_create(device, C.byref(h))
        if rc != GD_OK:
            raise GeoDockError(rc, self._lib.gd_last_error(None).decode())
        self._h = h
        self._batch = None
        self._K = 1

    def close(self):
        if getattr(self, "_h", None):
            self._lib.gd_destroy(self._h)
            self._h = None

    __del__ = close

    def _check(self, rc: int):
        if rc != GD_OK:
            raise GeoDockError(rc, self._lib.gd_last_error(self._h).decode())

    def set_stream(self, stream_ptr: int | None):
        self._check(self._lib.gd_set_stream(self._h, C.c_void_p(stream_ptr or 0)))

    def set_pocket(self, xyz: np.ndarray):
        pts = np.ascontiguousarray(xyz, dtype=np.float64).reshape(-1, 3)
        self._check(self._lib.gd_set_pocket(self._h, _p(pts, _f64p), len(pts)))

    def pocket_info(self) -> dict:
        c = np.zeros(3)
        d = np.zeros(3, np.int32)
        h = C.c_double()
        n = C.c_int64()
        m = C.c_int32()
        self._check(self._lib.gd_pocket_info(self._h, _p(c, _f64p), _p(d, _i32p), C.byref(h),
                                             C.byref(n), C.byref(m)))
        out = {"centre": c, "dims": d, "voxel": h.value, "n_candidates": n.value,
               "max_candidates": m.value}
        lv = (gd_index_level * 2)()
        self._check(self._lib.gd_pocket_index_stats(self._h, lv))
        out["levels"] = [{"dims": list(x.dims), "voxel": x.voxel, "candidates": x.candidates,
                          "record_bytes": x.record_bytes, "list_bytes": x.list_bytes} for x in lv]
        out["index_bytes"] = sum(x.record_bytes + x.list_bytes for x in lv)
        fmt = self._lib.gd_pocket_index_format(self._h)
        self._check(min(fmt, 0))
        out["format"] = "coded" if fmt == 1 else "fp64"
        return out

    def dock(self, batch: LigandBatch, knobs: Knobs, keep_poses: bool = False,
             out: "DockResult | None" = None, top_pose: bool = False) -> DockResult:
        """gd_dock_batch: host buffers in, host buffers out.  `out` (a
        DockResult of the right shape) is reused instead of allocating;
        top_pose fetches each ligand's top-1 final pose."""
        K = knobs.slots
        A = int(batch.atom_offsets[-1])
        res = out if out is not None and out.fits(batch.n_ligands, K, A, keep_poses, top_pose) \
            else DockResult.empty(batch.n_ligands, K, A, keep_poses, top_pose)
        b, k, r = batch.c_struct(), knobs.c_struct(), res.c_struct()
        self._check(self._lib.gd_dock_batch(self._h, C.byref(b), C.byref(k), C.byref(r)))
        self._batch = batch
        return res

    def upload(self, batch: LigandBatch):
        b = batch.c_struct()
        self._check(self._lib.gd_upload(self._h, C.byref(b)))
        self._batch = batch

    def dock_resident(self, knobs: Knobs, keep_poses: bool = False, top_pose: bool = False):
        k = knobs.c_struct()
        if keep_poses:
            k.flags |= GD_FLAG_KEEP_POSES
        if top_pose:
            k.flags |= GD_FLAG_TOP_POSE
        self._check(self._lib.gd_dock_resident(self._h, C.byref(k)))
        self._K = knobs.slots

    def download(self, result: DockResult):
        r = result.c_struct()
        self._check(self._lib.gd_download(self._h, C.byref(r)))
        return result

    def device_results(self) -> dict:
        """Device views (torch tensors, no copy) of the last resident dock's
        final-order table: final_score/orientation/seed_rank/evaluations [L, K]."""
        import torch
        d = gd_device_result()
        self._check(self._lib.gd_device_results(self._h, C.byref(d)))
        shape = (d.n_ligands, d.top_k)
        view = lambda ptr, ts, sh=shape: torch.as_tensor(_CudaArray(ptr, sh, ts), device="cuda")
        per_lig = (d.n_ligands,)
        return {"final_score": view(d.final_score, "<f8"), "orientation": view(d.orientation, "<i4"),
                "seed_rank": view(d.seed_rank, "<i4"), "evaluations": view(d.evaluations, "<i8"),
                "rigid_score": view(d.rigid_score, "<f8"),
                "feasibility_checks": view(d.feasibility_checks, "<i8"),
                "k_eff": view(d.k_eff, "<i4", per_lig), "poses_scored": view(d.poses_scored, "<i8", per_lig),
                "status": view(d.status, "<i4", per_lig)}

    def work_counters(self) -> dict:
        """Executed work of the last call made with GD_FLAG_COUNT_WORK."""
        out = (C.c_uint64 * 16)()
        self._check(self._lib.gd_work_counters(self._h, out))
        return {"rigid": dict(zip(WORK_FIELDS, out[0:7])), "flex": dict(zip(WORK_FIELDS, out[8:15]))}

    def phase_clocks(self) -> list:
        """Flex-kernel SM cycles per phase (GD_PHASE_CLOCKS builds; zeros otherwise)."""
        out = (C.c_uint64 * 16)()
        self._check(self._lib.gd_phase_clocks(self._h, out))
        return list(out)

    def rotation_profiles(self, batch: "LigandBatch | None" = None, flags: int = 0,
                          out: "ProfileBuffers | None" = None) -> "Profiles":
        """rotation_profile (analysis.hpp:37-56) of every fragment of `batch`
        (uploaded first) or of the batch staged last, from its poses.  `out`
        (ProfileBuffers.for_batch) reuses host output buffers across calls."""
        if batch is not None:
            self.upload(batch)
        staged = self._batch
        if staged is None:
            raise GeoDockError(GD_ERR_INVALID, "rotation_profiles: no batch staged")
        L = staged.n_ligands
        buf = out if out is not None and out.fits(staged) else ProfileBuffers.for_batch(staged)
        self._check(self._lib.gd_rotation_profiles(
            self._h, flags, _p(buf.scores, C.POINTER(C.c_double)),
            _p(buf.valid, C.POINTER(C.c_uint8)), _p(buf.rel, C.POINTER(C.c_double)),
            _p(buf.offs, C.POINTER(C.c_int32)), _p(buf.status, C.POINTER(C.c_int32)),
            len(buf.rel)))
        F = int(buf.offs[L])
        return Profiles(buf.scores[:F], buf.valid[:F].view(bool), buf.rel[:F], buf.offs[:L + 1],
                        buf.status[:L])

    # -- fine-grained drop-in entry points (one caller fragment per ligand) --
    @staticmethod
    def _fragset(batch: LigandBatch, membership, axis, anchor):
        mem = np.ascontiguousarray(membership, dtype=np.uint8).reshape(-1)
        ax = np.ascontiguousarray(np.atleast_1d(axis), dtype=np.int32)
        an = np.ascontiguousarray(np.atleast_1d(anchor), dtype=np.int32)
        assert len(mem) == batch.atom_offsets[-1] and len(ax) == len(an) == batch.n_ligands
        keep = (mem, ax, an)
        return gd_fragment_set(_p(mem, _u8p), _p(ax, _i32p), _p(an, _i32p)), keep

    def optimize_fragment(self, batch: LigandBatch, membership, axis, anchor, step: int,
                          refined: bool = False, entry_score=None) -> dict:
        """gd_optimize_fragment_batch: optimize_fragment_flat/_refined
        (kernel.hpp:125-198) of each ligand's fragment from its pose."""
        L, A = batch.n_ligands, int(batch.atom_offsets[-1])
        fs, keep = self._fragset(batch, membership, axis, anchor)
        out = {"best_angle": np.zeros(L, np.int32), "best_score": np.zeros(L),
               "evaluations": np.zeros(L, np.int64), "feasibility_checks": np.zeros(L, np.int64),
               "pose": np.zeros((A, 3)), "status": np.zeros(L, np.int32)}
        es = None if entry_score is None else np.ascontiguousarray(entry_score, dtype=np.float64)
        b = batch.c_struct()
        self._check(self._lib.gd_optimize_fragment_batch(
            self._h, C.byref(b), C.byref(fs), step, int(bool(refined)), _p(es, _f64p),
            _p(out["best_angle"], _i32p), _p(out["best_score"], _f64p),
            _p(out["evaluations"], _i64p), _p(out["feasibility_checks"], _i64p),
            _p(out["pose"], _f64p), _p(out["status"], _i32p)))
        self._batch = None
        return out

    def rotate_fragment(self, batch: LigandBatch, membership, axis, anchor, angles):
        """gd_rotate_fragment_batch (rotate_fragment_into, geometry.hpp:161-186)."""
        L, A = batch.n_ligands, int(batch.atom_offsets[-1])
        fs, keep = self._fragset(batch, membership, axis, anchor)
        ang = np.ascontiguousarray(np.atleast_1d(angles), dtype=np.float64)
        pose, status = np.zeros((A, 3)), np.zeros(L, np.int32)
        b = batch.c_struct()
        self._check(self._lib.gd_rotate_fragment_batch(self._h, C.byref(b), C.byref(fs),
                                                       _p(ang, _f64p), _p(pose, _f64p),
                                                       _p(status, _i32p)))
        self._batch = None
        return pose, status

    def check_bumps(self, batch: LigandBatch, membership, axis, anchor):
        """gd_check_bumps_batch (check_bumps, geometry.hpp:199-213)."""
        L = batch.n_ligands
        fs, keep = self._fragset(batch, membership, axis, anchor)
        feas, status = np.zeros(L, np.uint8), np.zeros(L, np.int32)
        b = batch.c_struct()
        self._check(self._lib.gd_check_bumps_batch(self._h, C.byref(b), C.byref(fs),
                                                   _p(feas, _u8p), _p(status, _i32p)))
        self._batch = None
        return feas.astype(bool), status

    def ligand_error(self, l: int) -> str:
        buf = C.create_string_buffer(512)
        self._check(self._lib.gd_ligand_error(self._h, l, buf, 512))
        return buf.value.decode()

    def l2_gather_peak_gbs(self) -> float:
        g = C.c_double()
        self._check(self._lib.gd_l2_gather_peak(self._h, C.byref(g)))
        return g.value

    def l2_gather_rate_gbs(self, warps_per_sm: int) -> float:
        """gd_l2_gather_rate: one dependent random gather in flight per lane."""
        g = C.c_double()
        self._check(self._lib.gd_l2_gather_rate(self._h, warps_per_sm, C.byref(g)))
        return g.value

    def fp64_peak_tflops(self) -> float:
        t = C.c_double()
        self._check(self._lib.gd_fp64_peak(self._h, C.byref(t)))
        return t.value

    def timing(self) -> dict:
        t = gd_timing()
        self._check(self._lib.gd_last_timing(self._h, C.byref(t)))
        return {f: getattr(t, f) for f, _ in gd_timing._fields_}

    def overlap_scores(self, poses: np.ndarray, brute: bool = False) -> np.ndarray:
        """overlap_score (geometry.hpp:140) of poses shaped [n_poses, n_atoms, 3]."""
        p = np.ascontiguousarray(poses, dtype=np.float64)
        if p.ndim == 2:
            p = p[None]
        out = np.zeros(p.shape[0])
        self._check(self._lib.gd_overlap_score_batch(
            self._h, _p(p, _f64p), p.shape[1], p.shape[0],
            GD_FLAG_BRUTE_FORCE if brute else 0, _p(out, _f64p)))
        return out


class MultiDocker:
    """gd_multi: one process, several GPUs (or several contexts on one GPU),
    cost-weighted chunks pulled from a shared cursor."""

    def __init__(self, devices=None, n_devices: int = 0):
        self._lib = lib()
        h = C.c_void_p()
        if devices is not None:
            dv = np.ascontiguousarray(devices, dtype=np.int32)
            rc = self._lib.gd_multi_create(_p(dv, _i32p), len(dv), C.byref(h))
        else:
            rc = self._lib.gd_multi_create(None, n_devices, C.byref(h))
        if rc != GD_OK:
            raise GeoDockError(rc, self._lib.gd_multi_last_error(None).decode())
        self._h = h

    def close(self):
        if getattr(self, "_h", None):
            self._lib.gd_multi_destroy(self._h)
            self._h = None

    __del__ = close

    def _check(self, rc: int):
        if rc != GD_OK:
            raise GeoDockError(rc, self._lib.gd_multi_last_error(self._h).decode())

    @property
    def size(self) -> int:
        return int(self._lib.gd_multi_size(self._h))

    def set_pocket(self, xyz: np.ndarray):
        pts = np.ascontiguousarray(xyz, dtype=np.float64).reshape(-1, 3)
        self._check(self._lib.gd_multi_set_pocket(self._h, _p(pts, _f64p), len(pts)))

    def dock(self, batch: LigandBatch, knobs: Knobs, keep_poses: bool = False,
             out: "DockResult | None" = None, top_pose: bool = False) -> DockResult:
        K = knobs.slots
        A = int(batch.atom_offsets[-1])
        res = out if out is not None and out.fits(batch.n_ligands, K, A, keep_poses, top_pose) \
            else DockResult.empty(batch.n_ligands, K, A, keep_poses, top_pose)
        b, k, r = batch.c_struct(), knobs.c_struct(), res.c_struct()
        self._check(self._lib.gd_multi_dock_batch(self._h, C.byref(b), C.byref(k), C.byref(r)))
        return res

    def ligand_error(self, l: int) -> str:
        buf = C.create_string_buffer(512)
        self._check(self._lib.gd_multi_ligand_error(self._h, l, buf, 512))
        return buf.value.decode()

    def stats(self) -> list:
        out = (gd_multi_stats * self.size)()
        self._check(self._lib.gd_multi_last_stats(self._h, out, self.size))
        return [{"ligands": s.ligands, "chunks": s.chunks, "busy_ms": s.busy_ms} for s in out]


# ---------------------------------------------------------------------------
# Host helpers
# ---------------------------------------------------------------------------
def optimal_tile_size(step: int) -> int:
    return int(lib().gd_optimal_tile_size(step))


def fit_cost_model(features, times):
    """fit (perf_model.hpp:57-105) via gd_fit_cost_model: features [n, 3]
    (pocket points, avg atoms, avg rotamers), times [n] s/ligand ->
    (coefficients [7], intercept, adjusted R^2)."""
    f = np.ascontiguousarray(features, dtype=np.float64).reshape(-1, 3)
    t = np.ascontiguousarray(times, dtype=np.float64)
    coef = np.zeros(7)
    icpt, r2 = C.c_double(), C.c_double()
    msg = C.create_string_buffer(512)
    rc = lib().gd_fit_cost_model(_p(f, _f64p), _p(t, _f64p), len(t), _p(coef, _f64p),
                                 C.byref(icpt), C.byref(r2), msg, 512)
    if rc != GD_OK:
        raise GeoDockError(rc, msg.value.decode())
    return coef, icpt.value, r2.value


def ligand_graph(xyz, radii, bonds, rotatable):
    """Native find_rotamers + grow_fragments (gd_ligand_graph): returns
    (rotamer bond indices [R], membership [2R, n] bool: row 2r = left), or
    raises GeoDockError with the Ligand validation message."""
    x = np.ascontiguousarray(xyz, dtype=np.float64).reshape(-1, 3)
    r = np.ascontiguousarray(radii, dtype=np.float64)
    b = np.ascontiguousarray(bonds, dtype=np.int32).reshape(-1, 2)
    ro = np.ascontiguousarray(rotatable, dtype=np.uint8)
    n, nb = len(x), len(b)
    rb = np.zeros(max(nb, 1), np.int32)
    mem = np.zeros((max(2 * nb, 1), max(n, 1)), np.uint8)
    cnt = C.c_int32()
    msg = C.create_string_buffer(256)
    rc = lib().gd_ligand_graph(n, _p(x, _f64p), _p(r, _f64p), nb, _p(b, _i32p), _p(ro, _u8p),
                               C.byref(cnt), _p(rb, _i32p), _p(mem, _u8p), msg, 256)
    if rc != GD_OK:
        raise GeoDockError(GD_ERR_INVALID, msg.value.decode())
    k = cnt.value
    return rb[:k].copy(), mem[:2 * k, :n].astype(bool)


def orientations(step: int):
    n = lib().gd_orientations(step, None, None, 0)
    if n < 0:
        raise GeoDockError(GD_ERR_INVALID, "rigid step must divide 360")
    idx = np.zeros(n, np.int32)
    R = np.zeros((n, 9))
    lib().gd_orientations(step, _p(idx, _i32p), _p(R, _f64p), n)
    return idx, R.reshape(n, 3, 3)


_synth_override = None


def set_synth_library(path) -> None:
    """Generate synthetic inputs with the gd_synth_* functions of another
    library built from the same csrc/synth.cpp (oracle/libgd_synth.so): the
    reference benchmark arm builds its inputs without the product library."""
    global _synth_override
    h = C.CDLL(str(path))
    for name in ("gd_synth_pocket", "gd_synth_ligand_size", "gd_synth_ligand"):
        res, args = SIGNATURES[name]
        getattr(h, name).restype = res
        getattr(h, name).argtypes = args
    _synth_override = h


def _synth() -> C.CDLL:
    return _synth_override if _synth_override is not None else lib()


def synth_pocket(a: float, b: float, c: float, spacing: float, rough_max: float = 0.0,
                 seed: int = 0) -> np.ndarray:
    n = _synth().gd_synth_pocket(a, b, c, spacing, rough_max, seed, None, 0)
    out = np.zeros((n, 3))
    _synth().gd_synth_pocket(a, b, c, spacing, rough_max, seed, _p(out, _f64p), n)
    return out


def synth_ligands(base_seed: int, ids, n_lo: int = 20, n_hi: int = 60, fixed_n: int = 0,
                  r_cap: int = 12, fixed_r: int = -1, centre=(0.0, 0.0, 0.0)) -> LigandBatch:
    """BASELINE random-walk-tree ligands `ids` of the family `base_seed`."""
    L = _synth()
    ids = list(ids)
    sizes = np.zeros(len(ids), np.int32)
    tmp = C.c_int32()
    for i, lid in enumerate(ids):
        if L.gd_synth_ligand_size(base_seed, lid, n_lo, n_hi, fixed_n, C.byref(tmp)) != GD_OK:
            raise GeoDockError(GD_ERR_INVALID, "bad ligand size range")
        sizes[i] = tmp.value
    ao = np.zeros(len(ids) + 1, np.int32)
    ao[1:] = np.cumsum(sizes)
    bo = np.zeros(len(ids) + 1, np.int32)
    bo[1:] = np.cumsum(sizes - 1)
    xyz = np.zeros((ao[-1], 3))
    radii = np.zeros(ao[-1])
    bonds = np.zeros((bo[-1], 2), np.int32)
    rot = np.zeros(bo[-1], np.uint8)
    cen = np.ascontiguousarray(centre, dtype=np.float64)
    for i, lid in enumerate(ids):
        a0, b0 = ao[i], bo[i]
        rc = L.gd_synth_ligand(base_seed, lid, n_lo, n_hi, fixed_n, r_cap, fixed_r, _p(cen, _f64p),
                               _p(xyz[a0:], _f64p), _p(radii[a0:], _f64p), _p(bonds[b0:], _i32p),
                               _p(rot[b0:], _u8p))
        if rc < 0:
            raise GeoDockError(GD_ERR_INVALID, "ligand synthesis failed")
    return LigandBatch(ao, xyz, radii, bo, bonds, rot)
