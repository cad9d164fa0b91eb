"""Ligand preprocessing on the GPU (csrc/prep.cu) against the reference's
Ligand constructor / find_rotamers / grow_fragments (molecule.hpp:66-301).

The search kernels read only what prep.cu writes, so docking results
bit-exact with the CPU oracle pin the far masks, rotamer order and
fragments; these cases aim at the graph corners: every rejection rule,
rings (a rotatable ring bond is not a bridge, so no rotamer), more than 32
rotamers (several lane rounds), more than 64 atoms (several mask words),
duplicate bonds in either orientation, and atom counts rejected up front.
"""
import numpy as np
import pytest

from paper_1901_06363_b200 import Knobs, LigandBatch, workloads as W
from gd_test_helpers import Lig, assert_same_result

pytestmark = pytest.mark.gpu


def _zigzag(n, dz=0.0):
    """A self-avoiding zig-zag chain, 1.5 A bonds."""
    return [[1.3 * i, 0.75 * (i % 2), dz] for i in range(n)]


def _ring_ligand():
    """A hexagon (every ring bond flagged rotatable) with a 4-atom tail
    whose non-terminal bonds are real rotamers."""
    hexa = [[1.5 * np.cos(k * np.pi / 3), 1.5 * np.sin(k * np.pi / 3), 0.0] for k in range(6)]
    tail = [[3.0 + 1.3 * i, 0.75 * (i % 2), 0.0] for i in range(4)]
    bonds = [(k, (k + 1) % 6, True) for k in range(6)] + [(0, 6, True), (6, 7, True), (7, 8, True),
                                                          (8, 9, True)]
    return Lig(hexa + tail, bonds, radius=1.1)


def _fused_rings():
    """Two fused rings plus a ring-to-chain bridge: only the bridge and the
    chain bonds are rotamers; the bonds are listed high-index first."""
    pos = [[0, 0, 0], [1.5, 0, 0], [2.2, 1.3, 0], [1.5, 2.6, 0], [0, 2.6, 0], [-0.7, 1.3, 0],
           [3.7, 1.3, 0], [5.0, 2.0, 0], [6.3, 1.3, 0], [7.6, 2.0, 0]]
    bonds = [(1, 0, True), (2, 1, True), (3, 2, True), (4, 3, True), (5, 4, True), (0, 5, True),
             (5, 2, True), (6, 2, True), (7, 6, True), (8, 7, True), (9, 8, False)]
    return Lig(pos, bonds, radius=1.0)


def test_graph_corners_dock_exactly(docker):
    O = pytest.importorskip("oracle.oracle_py")
    pocket = W.config(1).pocket()
    c = pocket.mean(axis=0)
    long = Lig(_zigzag(80), [(i, i + 1, True) for i in range(79)], radius=0.9)       # 77 rotamers, 2 words
    huge = Lig(_zigzag(200), [(i, i + 1, i % 3 == 0) for i in range(199)], radius=0.9)  # 4 words
    parts = [_ring_ligand(), _fused_rings(), long, huge]
    batch = LigandBatch.from_parts([(p.xyz + c - p.xyz.mean(axis=0), p.radii, p.bonds, p.rot)
                                    for p in parts])
    docker.set_pocket(pocket)
    for knobs in (Knobs(90, 90, 0.0, 1, False), Knobs.baseline(90, 60, 1, 3)):
        got = docker.dock(batch, knobs, keep_poses=True)
        want = O.dock_batch(batch, pocket, knobs, nthreads=O.threads())
        assert (got.status == 0).all()
        assert_same_result(got, want)


def test_every_rejection_rule(docker):
    """Each invalid ligand is skipped with the reference's message; its
    neighbours in the batch dock normally."""
    O = pytest.importorskip("oracle.oracle_py")
    good = Lig(_zigzag(6), [(i, i + 1, True) for i in range(5)])
    nan = good.xyz.copy()
    nan[2, 1] = np.nan
    cases = {
        "self-bond": Lig(_zigzag(4), [(0, 1, True), (1, 1, False), (2, 3, True)]),
        "bond index out of range": Lig(_zigzag(4), [(0, 1, True), (1, 2, True), (2, 7, False)]),
        "duplicate bond": Lig(_zigzag(4), [(0, 1, True), (1, 2, True), (2, 1, False), (2, 3, True)]),
        "non-positive radius": Lig(_zigzag(4), [(0, 1, True), (1, 2, True), (2, 3, True)],
                                   radius=[1.0, 1.0, 0.0, 1.0]),
        "non-finite position": Lig(nan, [(i, i + 1, True) for i in range(5)]),
        "disconnected": Lig(_zigzag(5), [(0, 1, True), (1, 2, True), (3, 4, True)]),
        "needs at least 2 atoms": Lig([[0, 0, 0]], []),
        "more than 4096 atoms is not supported": Lig(_zigzag(4097), [(i, i + 1, False) for i in range(4096)]),
    }
    parts = [good]
    for lig in cases.values():
        parts += [lig, good]
    batch = LigandBatch.from_parts([p.args for p in parts])
    pocket = W.config(0).pocket()
    docker.set_pocket(pocket)
    knobs = Knobs.baseline(90, 60, 1, 2)
    for path in ("batch", "resident"):
        if path == "batch":
            got = docker.dock(batch, knobs)
        else:
            from paper_1901_06363_b200 import DockResult
            docker.upload(batch)
            docker.dock_resident(knobs)
            got = docker.download(DockResult.empty(batch.n_ligands, knobs.slots,
                                                   int(batch.atom_offsets[-1]), False))
        for i, what in enumerate(cases):
            l = 2 * i + 1
            assert got.status[l] == 1 and got.k_eff[l] == 0, (path, what)
            assert what in docker.ligand_error(l), (path, what, docker.ligand_error(l))
        assert (got.status[0::2] == 0).all()
    keep = [l for l in range(batch.n_ligands) if l % 2 == 0]
    sub = batch.subset(keep)
    want = O.dock_batch(sub, pocket, knobs, nthreads=1, keep_poses=False)
    for f in ("final_score", "orientation", "evaluations", "feasibility_checks"):
        assert np.array_equal(getattr(got, f)[keep], getattr(want, f)), f


def test_top_pose_is_slot_zero_pose(docker):
    """gd_result.top_pose (each ligand's top-1 final pose, what the e2e bench
    fetches) equals slot 0 of the full pose table, through gd_dock_batch, the
    resident path (GD_FLAG_TOP_POSE) and gd_multi; skipped ligands read 0."""
    from paper_1901_06363_b200 import DockResult, MultiDocker
    w = W.config(1)
    pocket = w.pocket()
    batch = w.ligands(range(600))
    batch.radii[batch.atom_offsets[7]] = 0.0  # ligand 7 is rejected
    docker.set_pocket(pocket)
    full = docker.dock(batch, w.knobs, keep_poses=True)
    K = w.knobs.slots
    want = np.zeros((int(batch.atom_offsets[-1]), 3))
    for l in range(batch.n_ligands):
        if full.status[l] == 0:
            a0, a1 = batch.atom_offsets[l], batch.atom_offsets[l + 1]
            want[a0:a1] = full.pose(batch, l, 0)
    assert full.status[7] == 1
    got = docker.dock(batch, w.knobs, top_pose=True)
    assert np.array_equal(got.top_pose, want)
    assert np.array_equal(got.final_score, full.final_score)
    docker.upload(batch)
    docker.dock_resident(w.knobs, top_pose=True)
    res = docker.download(DockResult.empty(batch.n_ligands, K, int(batch.atom_offsets[-1]), False, True))
    assert np.array_equal(res.top_pose, want)
    m = MultiDocker([0, 0])
    try:
        m.set_pocket(pocket)
        mres = m.dock(batch, w.knobs, top_pose=True)
        assert np.array_equal(mres.top_pose, want)
    finally:
        m.close()


def test_bond_count_far_above_atom_count(docker):
    """Shared memory is sized by atoms, not bonds: a 24-atom ligand with
    every one of its 276 atom pairs bonded (all flagged rotatable, none a
    bridge) docks with no rotamers, and one with each bond listed twice
    (552 bonds) is rejected as a duplicate -- neither fails the batch."""
    O = pytest.importorskip("oracle.oracle_py")
    n = 24
    pos = [[1.6 * np.cos(2 * np.pi * k / n) * (1 + 0.3 * (k % 3)), 1.6 * np.sin(2 * np.pi * k / n),
            0.4 * (k % 5)] for k in range(n)]
    pairs = [(a, b) for a in range(n) for b in range(a + 1, n)]
    dense = Lig(pos, [(a, b, True) for a, b in pairs], radius=0.5)
    dup = Lig(pos, [(a, b, True) for a, b in pairs] + [(b, a, False) for a, b in pairs], radius=0.5)
    chain = Lig(_zigzag(8), [(i, i + 1, True) for i in range(7)])
    batch = LigandBatch.from_parts([dense.args, dup.args, chain.args])
    pocket = W.config(0).pocket()
    c = pocket.mean(axis=0)
    batch.xyz[:] += c - batch.xyz.mean(axis=0)
    docker.set_pocket(pocket)
    knobs = Knobs.baseline(90, 60, 1, 2)
    got = docker.dock(batch, knobs, keep_poses=True)
    assert list(got.status) == [0, 1, 0]
    assert "duplicate bond" in docker.ligand_error(1)
    keep = [0, 2]
    want = O.dock_batch(batch.subset(keep), pocket, knobs, nthreads=1)
    for f in ("final_score", "orientation", "evaluations", "feasibility_checks"):
        assert np.array_equal(getattr(got, f)[keep], getattr(want, f)), f
