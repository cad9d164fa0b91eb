"""The two voxel-record formats of the exact nearest-point index (kernels.h):
fp64 records, and coded records (a candidate = three 16-bit offsets into the
pocket's table of distinct coordinate values) chosen by gd_set_pocket when
that table fits 128 entries -- every BASELINE pocket, since they are lattices.

Both must return the full scan's fp64 minimum bit for bit, so docking results
are identical across formats and identical to the reference (oracle/_ref).
GD_INDEX_COMPACT / GD_VOXEL_OVERFLOW are read per gd_set_pocket call; each
case uses a fresh context so the pocket cache cannot serve the other format.
"""
import contextlib
import os

import numpy as np
import pytest

from paper_1901_06363_b200 import workloads as W
from gd_test_helpers import assert_same_result

pytestmark = pytest.mark.gpu


@contextlib.contextmanager
def _env(**kv):
    old = {k: os.environ.get(k) for k in kv}
    os.environ.update({k: str(v) for k, v in kv.items()})
    try:
        yield
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


@contextlib.contextmanager
def _docker(pocket, fmt, overflow=1024):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1901_06363_b200 import Docker
    d = Docker(int(os.environ.get("GD_TEST_DEVICE", "0")))
    try:
        with _env(GD_INDEX_COMPACT=1 if fmt == "coded" else 0, GD_VOXEL_OVERFLOW=overflow):
            d.set_pocket(pocket)
        yield d
    finally:
        d.close()


def _dense_queries(pocket, n=60000, seed=11):
    rng = np.random.default_rng(seed)
    lo, hi = pocket.min(axis=0), pocket.max(axis=0)
    far = rng.uniform(lo - 36.0, hi + 36.0, size=(n, 3))
    near = rng.uniform(lo - 3.5, hi + 3.5, size=(n, 3))
    base = pocket[rng.integers(0, len(pocket), n)]
    ties = base + rng.choice([-0.5, 0.0, 0.5], size=(n, 3)) + rng.normal(0, 1e-9, (n, 3))
    exact_ties = base + rng.choice([-0.5, 0.0, 0.5], size=(n, 3))
    return np.concatenate([far, near, ties, exact_ties])[:, None, :]


def _pockets():
    w3 = W.config(3)
    by_size = sorted((W.pocket_of(w3, i) for i in range(16)), key=len)
    return {"c1": W.config(1).pocket(), "c3-smallest": by_size[0], "c3-largest": by_size[-1]}


@pytest.mark.parametrize("which", ["c1", "c3-smallest", "c3-largest"])
@pytest.mark.parametrize("overflow", [1024, 3])
def test_coded_index_minima_equal_full_scan(which, overflow):
    """Coded records on BASELINE pockets: exact minima on 240k one-atom
    queries (uniform, near field, lattice Voronoi boundaries).  overflow=3
    turns every voxel with more than 3 candidates into an overflow voxel,
    which walks the shared whole-pocket head (coded blocks of 5)."""
    pocket = _pockets()[which]
    q = _dense_queries(pocket)
    with _docker(pocket, "coded", overflow) as d:
        info = d.pocket_info()
        assert info["format"] == "coded"
        if overflow == 3:
            assert info["max_candidates"] == len(pocket)
        idx = d.overlap_scores(q)
        brute = d.overlap_scores(q, brute=True)
    bad = np.flatnonzero(idx != brute)
    assert bad.size == 0, (bad[:5], q[bad[:5], 0])


def test_coded_index_is_smaller_and_chosen_only_for_small_tables():
    pocket = W.config(1).pocket()
    with _docker(pocket, "coded") as d:
        coded = d.pocket_info()
    with _docker(pocket, "fp64") as d:
        fp64 = d.pocket_info()
    assert coded["format"] == "coded" and fp64["format"] == "fp64"
    # Same candidate sets, fewer list bytes (5 per 32-byte block, 4 inline).
    assert coded["n_candidates"] == fp64["n_candidates"]
    assert coded["index_bytes"] < fp64["index_bytes"]
    # An off-lattice pocket has too many distinct coordinates: fp64 records.
    rng = np.random.default_rng(3)
    with _docker(rng.uniform(-8, 8, size=(500, 3)), "coded") as d:
        assert d.pocket_info()["format"] == "fp64"
    # Lattice pockets with up to 128 distinct values in total stay coded.
    g = np.mgrid[-20:21, -20:21, -20:21].reshape(3, -1).T.astype(float) * 0.5
    lat = g[(g ** 2).sum(1) <= 100.0]
    with _docker(lat, "coded") as d:
        assert d.pocket_info()["format"] == "coded"


@pytest.mark.parametrize("overflow", [1024, 2])
def test_docking_identical_across_formats_and_to_reference(overflow):
    """48 config-1 ligands (rigid sweep, fragment searches, top-K) docked on
    both formats: every result field bit-identical, and equal to the
    reference compiled from its own sources (oracle/_ref) when present."""
    from oracle import oracle_py as O
    w = W.config(1)
    pocket = w.pocket()
    batch = w.ligands(range(48))
    with _docker(pocket, "coded", overflow) as d:
        assert d.pocket_info()["format"] == "coded"
        a = d.dock(batch, w.knobs, keep_poses=True)
    with _docker(pocket, "fp64", overflow) as d:
        b = d.dock(batch, w.knobs, keep_poses=True)
    assert_same_result(a, b, ctx="coded vs fp64: ")
    if overflow == 1024:
        impl = "ref" if O.have_ref() else "oracle"
        want = O.dock_batch(batch, pocket, w.knobs, nthreads=O.threads(),
                            **({"impl": "ref"} if impl == "ref" else {}))
        assert_same_result(a, want, ctx=f"coded vs {impl}: ")


def test_coded_profiles_and_fragment_api_identical():
    """The rotation-profile kernel and the fine-grained fragment search read
    the index too: identical across formats."""
    from test_gpu_fragment_api import _batch, _c1_ligands, _items
    w = W.config(1)
    pocket = w.pocket()
    batch = w.ligands(range(24))
    ligs, _ = _c1_ligands(8)
    items = _items(ligs)[:40]
    prof, frag = {}, {}
    for fmt in ("coded", "fp64"):
        with _docker(pocket, fmt) as d:
            pr = d.rotation_profiles(batch)
            prof[fmt] = (pr.scores.copy(), pr.valid.copy())
            fb, mem, ax, an = _batch(items)
            frag[fmt] = d.optimize_fragment(fb, mem, ax, an, 10)
    assert np.array_equal(prof["coded"][0], prof["fp64"][0])
    assert np.array_equal(prof["coded"][1], prof["fp64"][1])
    for k in frag["coded"]:
        assert np.array_equal(frag["coded"][k], frag["fp64"][k]), k
