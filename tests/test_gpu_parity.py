"""GPU parity: the CUDA path through the C-ABI against the CPU oracle.

Bar: bit-exact.  Every score is fp64 computed with the reference's
expression trees, so top-K orientation indices, ordering, scores, counters
and final coordinates must be identical -- stricter than BASELINE's 1e-4
relative tolerance on scores/coordinates, which we therefore also meet.
"""
import numpy as np
import pytest

from paper_1901_06363_b200 import Knobs, workloads as W
from gd_test_helpers import assert_same_result

pytestmark = pytest.mark.gpu

REL_TOL = 1e-4  # BASELINE.json north_star tolerance (we require bit-exact)


def _oracle():
    from oracle import oracle_py
    return oracle_py


def _cpu(batch, pocket, knobs):
    """The reference itself (oracle/_ref, PocketIndex) when built, else the C oracle."""
    O = _oracle()
    if O.have_ref():
        return O.dock_batch(batch, pocket, knobs, nthreads=O.threads(), impl="ref")
    return O.dock_batch(batch, pocket, knobs, nthreads=O.threads())


def test_config0_full_parity(docker):
    w = W.config(0)
    pocket = w.pocket()
    batch = w.ligands()
    docker.set_pocket(pocket)
    got = docker.dock(batch, w.knobs, keep_poses=True)
    want = _oracle().dock_batch(batch, pocket, w.knobs, nthreads=1)
    assert got.k_eff[0] == 30
    assert_same_result(got, want)
    np.testing.assert_allclose(got.final_score, want.final_score, rtol=REL_TOL)


def test_config0_brute_force_equals_index(docker):
    w = W.config(0)
    docker.set_pocket(w.pocket())
    batch = w.ligands()
    a = docker.dock(batch, w.knobs, keep_poses=True)
    k = Knobs(**{**w.knobs.__dict__, "flags": 1})
    b = docker.dock(batch, k, keep_poses=True)
    assert_same_result(a, b)


@pytest.mark.parametrize("n_lig", [48])
def test_config1_subset_parity(docker, n_lig):
    w = W.config(1)
    pocket = w.pocket()
    batch = w.ligands(range(n_lig))
    docker.set_pocket(pocket)
    got = docker.dock(batch, w.knobs, keep_poses=True)
    want = _cpu(batch, pocket, w.knobs)
    assert_same_result(got, want)


def test_pipelined_dock_batch_equals_resident_path(docker):
    """gd_dock_batch splits >1024-ligand batches into chunks on two streams;
    it must equal the single-launch resident path bit for bit, and the
    reference on ligands at the chunk boundaries."""
    from paper_1901_06363_b200 import DockResult
    w = W.config(1)
    pocket = w.pocket()
    batch = w.ligands(range(2600))
    docker.set_pocket(pocket)
    got = docker.dock(batch, w.knobs, keep_poses=True)
    docker.upload(batch)
    docker.dock_resident(w.knobs, keep_poses=True)
    want = docker.download(DockResult.empty(batch.n_ligands, w.knobs.slots,
                                            int(batch.atom_offsets[-1]), True))
    assert_same_result(got, want)
    picks = [0, 1299, 1300, 2599]
    sub = batch.subset(picks)
    ref = _cpu(sub, pocket, w.knobs)
    for i, l in enumerate(picks):
        assert np.array_equal(got.orientation[l], ref.orientation[i])
        assert np.array_equal(got.final_score[l], ref.final_score[i])
        assert np.array_equal(got.evaluations[l], ref.evaluations[i])


def test_device_results_views_match_download(docker):
    """gd_device_results: zero-copy torch views of the resident top-K table
    (what the multi-GPU gather all-gathers) equal gd_download's copy."""
    from paper_1901_06363_b200 import DockResult
    w = W.config(1)
    pocket = w.pocket()
    batch = w.ligands(range(300))
    docker.set_pocket(pocket)
    docker.upload(batch)
    docker.dock_resident(w.knobs)
    host = docker.download(DockResult.empty(batch.n_ligands, w.knobs.slots,
                                            int(batch.atom_offsets[-1]), False))
    dev = docker.device_results()
    from paper_1901_06363_b200.sharding import DeviceGather
    for f in DeviceGather.FIELDS:  # every gd_result field but the poses, empty slots included
        assert np.array_equal(dev[f].cpu().numpy(), getattr(host, f)), f
    # The bench's N>1 gather over those views (a world-1 NCCL group here).
    import socket
    import torch.distributed as dist
    from paper_1901_06363_b200.sharding import DeviceGather
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1)
    try:
        out = DeviceGather(dev, 1)()
        for f in DeviceGather.FIELDS:
            assert np.array_equal(out[f][0].cpu().numpy(), getattr(host, f)), f
    finally:
        dist.destroy_process_group()


def test_device_results_empty_slots_and_failed_ligands(docker):
    """The device table carries the host's empty-slot values: K = 40 above a
    24-orientation grid (rigid 90), and a ligand the validation rejects."""
    from paper_1901_06363_b200 import DockResult, Knobs
    from paper_1901_06363_b200.sharding import DeviceGather
    w = W.config(1)
    pocket = w.pocket()
    batch = w.ligands(range(12))
    batch.radii[batch.atom_offsets[5]] = -1.0  # ligand 5: "non-positive radius on atom 0"
    knobs = Knobs.baseline(90, 60, 1, 40)
    docker.set_pocket(pocket)
    docker.upload(batch)
    docker.dock_resident(knobs)
    host = docker.download(DockResult.empty(batch.n_ligands, knobs.slots,
                                            int(batch.atom_offsets[-1]), False))
    assert host.status[5] != 0 and (host.status[np.arange(12) != 5] == 0).all()
    assert (host.k_eff[host.status == 0] < 40).all() and (host.orientation[:, -1] == -2).all()
    dev = docker.device_results()
    for f in DeviceGather.FIELDS:
        assert np.array_equal(dev[f].cpu().numpy(), getattr(host, f)), f


def test_config2_knobs_parity(docker):
    """c2 knobs (rigid 10, frag 10, 3 restarts, K=100) on two c1-distribution ligands."""
    w = W.config(2)
    pocket = w.pocket()
    batch = w.ligands([3, 11])
    docker.set_pocket(pocket)
    got = docker.dock(batch, w.knobs, keep_poses=True)
    want = _cpu(batch, pocket, w.knobs)
    assert (got.k_eff == 100).all()
    assert_same_result(got, want)


@pytest.mark.parametrize("top_k", [1, 32, 33, 64, 207, 208, 250])
def test_topk_sizes(docker, top_k):
    """Both top-K kernels (warp registers for K <= 32, rank merge above),
    including K >= #orientations (208 at 45 degrees: K = all of them)."""
    w = W.config(1)
    pocket = w.pocket()
    batch = w.ligands(range(4))
    knobs = Knobs.baseline(45, 90, 1, top_k)
    docker.set_pocket(pocket)
    got = docker.dock(batch, knobs, keep_poses=False)
    want = _cpu(batch, pocket, knobs)
    assert (got.k_eff == min(top_k, 208)).all()
    assert_same_result(got, want, poses=False)


@pytest.mark.parametrize("knobs", [
    Knobs(1, 45, 0.0, 1, False),    # Algorithm-1 baseline (test_kernel.cpp:241-250)
    Knobs(2, 90, 0.3, 2, True),     # determinism test config (test_kernel.cpp:205-220)
    Knobs(5, 90, 0.3, 1, False),    # screening invariance config (test_screening.cpp:45)
    Knobs(3, 45, 0.2, 1, True),     # spatial-index config (test_kernel.cpp:252-263)
    Knobs(10, 90, 0.5, 1, False),   # bookkeeping config (test_screening.cpp:62)
    Knobs(1, 90, 1.0, 1, False),    # threshold 1: every fragment at the low step
    Knobs(360, 360, 0.0, 3, False), # step 360: only the current pose
])
def test_given_pose_match_probes_shape(docker, knobs):
    """rigid_step 0 = the reference's screen path: match_probes_shape on the input pose."""
    O = _oracle()
    pocket, batch = None, None
    if O.have_ref():
        pocket, batch = O.ref_generate_synthetic(24, 4242)
    else:
        w = W.config(1)
        pocket = w.pocket()
        batch = w.ligands(range(24))
    docker.set_pocket(pocket)
    got = docker.dock(batch, knobs, keep_poses=True)
    want = O.dock_batch(batch, pocket, knobs, nthreads=O.threads())
    assert_same_result(got, want)


def test_large_ligands_multiword_masks(docker):
    """Ligands of 65..153 atoms (2-3 mask words) with many rotamers, from the
    reference's own generator envelope (synthetic.hpp DatasetSpec defaults)."""
    O = _oracle()
    if not O.have_ref():
        pytest.skip("oracle/_ref not built")
    pocket, batch = O.ref_generate_synthetic(6, 2718, 65, 153, 8, 30, 400, 10.0)
    assert batch.sizes.max() > 128
    docker.set_pocket(pocket)
    for knobs in (Knobs(30, 45, 0.0, 1, False), Knobs.baseline(45, 30, 1, 8),
                  Knobs(20, 45, 0.25, 2, True, 45, 4)):
        got = docker.dock(batch, knobs, keep_poses=True)
        want = O.dock_batch(batch, pocket, knobs, nthreads=O.threads(), impl="ref")
        assert_same_result(got, want)


def test_ligands_at_the_atom_limit(docker):
    """220-256 atoms (four mask words; the flex CTA narrows to fit shared
    memory) against the reference; 257 atoms takes the wide path
    (tests/test_gpu_wide.py) instead of being skipped."""
    from paper_1901_06363_b200 import LigandBatch, synth_ligands
    pocket = W.config(1).pocket()
    batch = synth_ligands(777, [0, 1], n_lo=220, n_hi=256, r_cap=12, centre=pocket.mean(axis=0))
    assert batch.sizes.min() >= 220 and batch.sizes.max() <= 256
    docker.set_pocket(pocket)
    knobs = Knobs(90, 90, 0.0, 1, False, 90, 3)
    got = docker.dock(batch, knobs, keep_poses=True)
    want = _cpu(batch, pocket, knobs)
    assert_same_result(got, want)
    n = 257
    xyz = np.stack([np.arange(n) * 1.5, np.zeros(n), np.zeros(n)], axis=1)
    big = LigandBatch.from_parts([(xyz, np.full(n, 1.2), np.stack([np.arange(n - 1), np.arange(1, n)], 1),
                                   np.zeros(n - 1, np.uint8))])
    res = docker.dock(big, knobs, keep_poses=True)
    assert res.status[0] == 0 and res.k_eff[0] == 3
    assert_same_result(res, _cpu(big, pocket, knobs))


def test_config3_rough_pocket(docker):
    """A config-3 pocket (random semi-axes, 1 A lattice, roughness mask)."""
    w = W.config(3)
    pocket = W.pocket_of(w, 5)
    batch = w.ligands(range(12), pocket.mean(axis=0))
    docker.set_pocket(pocket)
    got = docker.dock(batch, w.knobs, keep_poses=True)
    want = _cpu(batch, pocket, w.knobs)
    assert_same_result(got, want)


def test_edge_ligands(docker):
    """Two-atom rigid ligand, a ligand with no rotamers, an invalid ligand
    (disconnected) that must be skipped, and a single-point pocket."""
    from paper_1901_06363_b200 import LigandBatch
    from gd_test_helpers import Lig
    parts = [
        Lig([[0, 0, 0], [0, 0, 1.5]], [(0, 1, False)]),
        Lig([[0, 0, 0], [1.5, 0, 0], [3, 0.5, 0], [4.5, 0, 0]], [(0, 1, False), (1, 2, False), (2, 3, False)]),
        Lig([[0, 0, 0], [1.5, 0, 0], [9, 9, 9]], [(0, 1, True)]),  # disconnected
        Lig([[0, 0, 0], [0, 0, 1], [1, 0, 1], [1, 1, 1]], [(0, 1, True), (1, 2, True), (2, 3, True)]),
    ]
    batch = LigandBatch.from_parts([p.args for p in parts])
    O = _oracle()
    for pocket in (np.array([[0.5, 0.2, 0.1]]), W.config(0).pocket()):
        docker.set_pocket(pocket)
        for knobs in (Knobs.baseline(90, 30, 2, 5), Knobs(10, 45, 0.0, 1, True)):
            got = docker.dock(batch, knobs, keep_poses=True)
            want = O.dock_batch(batch, pocket, knobs, nthreads=1)
            assert got.status[2] == 1 and got.k_eff[2] == 0
            assert_same_result(got, want)


def test_overlap_score_kats(docker):
    """test_geometry.cpp:45-56 hand values through the GPU scoring kernel."""
    docker.set_pocket(np.array([[0.0, 0.0, 1.0]]))
    assert docker.overlap_scores(np.array([[0.0, 0.0, 0.0]]))[0] == 1.0
    docker.set_pocket(np.array([[0.0, 0.0, 0.0]]))
    assert docker.overlap_scores(np.array([[0.0, 0.0, 0.0], [0.0, 0.0, 3.0]]))[0] == 2.0 / (1e-12 + 9.0)
    docker.set_pocket(np.array([[0.0, 0.0, 1.0], [0.0, 0.0, 4.0]]))
    assert docker.overlap_scores(np.array([[0.0, 0.0, 2.0]]))[0] == 1.0


@pytest.mark.parametrize("which", ["c1", "c3-largest", "c3-smallest", "20k-points"])
def test_index_minimum_equals_full_scan_on_dense_queries(docker, which):
    """The (culled, brick-built) voxel index returns the full scan's fp64
    minimum for 300k single-atom queries: uniform over both grid levels and
    beyond them, plus points clustered on the pocket lattice's Voronoi
    boundaries (ties).  One-atom score = 1 / max(1e-12, min d^2), so equal
    scores are equal minima."""
    if which == "c1":
        pocket = W.config(1).pocket()
    elif which == "20k-points":  # beyond the culled build's 16,384 points: full-scan build
        g = np.mgrid[-21:22, -18:19, -15:16].reshape(3, -1).T.astype(float)
        pocket = g[(g[:, 0] / 21.0) ** 2 + (g[:, 1] / 18.0) ** 2 + (g[:, 2] / 15.0) ** 2 <= 1.0]
        assert len(pocket) > 16384
    else:
        w3 = W.config(3)
        pockets = sorted((W.pocket_of(w3, i) for i in range(16)), key=len)
        pocket = pockets[-1] if which == "c3-largest" else pockets[0]
    docker.set_pocket(pocket)
    rng = np.random.default_rng(11)
    lo, hi = pocket.min(axis=0), pocket.max(axis=0)
    far = rng.uniform(lo - 36.0, hi + 36.0, size=(100000, 3))
    near = rng.uniform(lo - 3.5, hi + 3.5, size=(100000, 3))
    # Half-integer offsets from lattice points: equidistant from neighbours.
    base = pocket[rng.integers(0, len(pocket), 100000)]
    ties = base + rng.choice([-0.5, 0.0, 0.5], size=(100000, 3)) + rng.normal(0, 1e-9, (100000, 3))
    q = np.concatenate([far, near, ties])[:, None, :]
    idx = docker.overlap_scores(q)
    brute = docker.overlap_scores(q, brute=True)
    bad = np.flatnonzero(idx != brute)
    assert bad.size == 0, (bad[:5], q[bad[:5], 0])


def test_overlap_scores_random_poses_exact(docker):
    """Index vs brute vs oracle on random poses, including far-away atoms."""
    O = _oracle()
    pocket = W.config(1).pocket()
    docker.set_pocket(pocket)
    rng = np.random.default_rng(7)
    poses = rng.uniform(-16, 16, size=(64, 40, 3))
    poses[0, 0] = [500.0, -300.0, 200.0]  # outside the grid: brute fallback
    idx = docker.overlap_scores(poses)
    brute = docker.overlap_scores(poses, brute=True)
    want = np.array([O.overlap_score(p, pocket) for p in poses])
    assert np.array_equal(idx, want)
    assert np.array_equal(brute, want)
