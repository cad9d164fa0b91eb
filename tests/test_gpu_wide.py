"""Ligands of more than 256 atoms: the reference docks any size
(molecule.hpp:66-89 has no limit), so the drop-in must too.  Up to 256 atoms
a chain is a warp with its state in shared memory; above, ligands are
preprocessed on the host (prep.cpp) and their chains run in
flex_wide_kernel, one CTA per chain with the state in HBM.  Everything is
compared bit-exact with the reference (oracle/_ref) or the C oracle:
top-K orientations and order, seed ranks, rigid and final scores, both
CandidateEvaluator counters and the final poses.
"""
import os

import numpy as np
import pytest

from paper_1901_06363_b200 import Knobs, LigandBatch, synth_ligands, workloads as W
from gd_test_helpers import Lig, assert_same_result

pytestmark = pytest.mark.gpu


def _cpu(batch, pocket, knobs):
    from oracle import oracle_py as O
    impl = "ref" if O.have_ref() else "oracle"
    return O.dock_batch(batch, pocket, knobs, nthreads=O.threads(), keep_poses=True, impl=impl)


def _parts(batch):
    ao, bo = batch.atom_offsets, batch.bond_offsets
    return [(batch.xyz[ao[l]:ao[l + 1]], batch.radii[ao[l]:ao[l + 1]], batch.bonds[bo[l]:bo[l + 1]],
             batch.rotatable[bo[l]:bo[l + 1]]) for l in range(batch.n_ligands)]


def _zigzag(n):
    return [[1.3 * i, 0.75 * (i % 2), 0.4 * ((i // 2) % 2)] for i in range(n)]


def _mixed(pocket):
    """c1 ligands interleaved with wide ones: 257 atoms (one over the warp
    path's limit), random-walk trees of 260-420 atoms, chains of 360 atoms
    (12 rotamers) and 1,000 atoms (16 mask words)."""
    c = pocket.mean(axis=0)
    small = _parts(W.config(1).ligands(range(5), c))
    trees = _parts(synth_ligands(4242, [0, 1, 2], n_lo=260, n_hi=420, r_cap=24, centre=c))
    edge = _parts(synth_ligands(4243, [0], fixed_n=257, r_cap=12, centre=c))
    chains = []
    for n, rot in ((360, lambda i: i % 29 == 3), (1000, lambda i: i in (200, 500, 800))):
        ch = Lig(_zigzag(n), [(i, i + 1, rot(i)) for i in range(n - 1)], radius=0.8)
        chains.append((ch.xyz + c - ch.xyz.mean(axis=0), ch.radii, ch.bonds, ch.rot))
    parts = [small[0], trees[0], small[1], edge[0], small[2], trees[1], chains[0], small[3], trees[2],
             chains[1], small[4]]
    return LigandBatch.from_parts(parts)


KNOBS = [
    Knobs(90, 90, 0.0, 1, False, 90, 3),       # flat, 3 candidates per search
    Knobs.baseline(90, 60, 2, 4),              # two restarts
    Knobs(30, 60, 0.2, 1, True, 90, 2),        # refined search above the threshold, flat below
]


@pytest.mark.parametrize("fmt", ["coded", "fp64"])
def test_wide_ligands_dock_exactly(docker, fmt):
    pocket = W.config(1).pocket()
    batch = _mixed(pocket)
    assert (batch.sizes > 256).sum() == 6 and batch.sizes.max() == 1000
    old = os.environ.get("GD_INDEX_COMPACT")
    os.environ["GD_INDEX_COMPACT"] = "1" if fmt == "coded" else "0"
    try:
        docker.set_pocket(pocket + (0.0 if fmt == "coded" else 1e-9))  # a new pocket: rebuild the index
        pk = pocket + (0.0 if fmt == "coded" else 1e-9)
        assert docker.pocket_info()["format"] == fmt
        for knobs in (KNOBS if fmt == "coded" else KNOBS[:1]):  # the CPU reference dominates the run time
            got = docker.dock(batch, knobs, keep_poses=True)
            assert (got.status == 0).all(), [docker.ligand_error(l) for l in range(batch.n_ligands)]
            want = _cpu(batch, pk, knobs)
            assert_same_result(got, want, ctx=f"{fmt} {knobs}: ")
    finally:
        if old is None:
            os.environ.pop("GD_INDEX_COMPACT", None)
        else:
            os.environ["GD_INDEX_COMPACT"] = old
        docker.set_pocket(pocket)


def test_wide_ligands_resident_given_pose_and_top_pose(docker):
    """The resident path (gd_upload + gd_dock_resident), the given-pose mode
    (rigid_step = 0, the reference screen's per-ligand call) and the top-1
    pose output agree with the batch path's full pose table."""
    pocket = W.config(1).pocket()
    batch = _mixed(pocket)
    docker.set_pocket(pocket)
    knobs = Knobs.baseline(90, 60, 1, 3)
    full = docker.dock(batch, knobs, keep_poses=True)
    top = docker.dock(batch, knobs, top_pose=True)
    for l in range(batch.n_ligands):
        a0, a1 = batch.atom_offsets[l], batch.atom_offsets[l + 1]
        assert np.array_equal(top.top_pose[a0:a1], full.pose(batch, l, 0)), l
    docker.upload(batch)
    docker.dock_resident(knobs, keep_poses=True)
    from paper_1901_06363_b200.native import DockResult
    res = docker.download(DockResult.empty(batch.n_ligands, knobs.slots, int(batch.atom_offsets[-1]), True))
    assert_same_result(res, full, ctx="resident: ")
    given = Knobs(60, 60, 0.0, 2, False)  # rigid_step 0: dock the given pose
    got = docker.dock(batch, given, keep_poses=True)
    assert_same_result(got, _cpu(batch, pocket, given), ctx="given pose: ")


def test_wide_ligand_rejections(docker):
    """Invalid wide ligands are skipped with the reference's message; the
    batch path's own size limit (4,096 atoms) has its own message."""
    pocket = W.config(1).pocket()
    c = pocket.mean(axis=0)
    ok = Lig(_zigzag(300), [(i, i + 1, i % 5 == 2) for i in range(299)], radius=0.8)
    cut = Lig(_zigzag(300), [(i, i + 1, True) for i in range(299) if i != 150], radius=0.8)
    dup = Lig(_zigzag(300), [(i, i + 1, True) for i in range(299)] + [(7, 6, False)], radius=0.8)
    huge = Lig(_zigzag(4097), [(i, i + 1, False) for i in range(4096)], radius=0.8)
    parts = [(x.xyz + c - x.xyz.mean(axis=0), x.radii, x.bonds, x.rot) for x in (ok, cut, dup, huge, ok)]
    batch = LigandBatch.from_parts(parts)
    docker.set_pocket(pocket)
    knobs = Knobs.baseline(90, 90, 1, 2)
    got = docker.dock(batch, knobs, keep_poses=True)
    assert got.status.tolist() == [0, 1, 1, 1, 0]
    assert got.k_eff.tolist() == [2, 0, 0, 0, 2]
    assert "disconnected ligand" in docker.ligand_error(1)
    assert "duplicate bond" in docker.ligand_error(2)
    assert "more than 4096 atoms is not supported" in docker.ligand_error(3)
    keep = batch.subset([0, 4])
    want = _cpu(keep, pocket, knobs)
    sub = docker.dock(keep, knobs, keep_poses=True)
    assert_same_result(sub, want)
    for f in ("orientation", "final_score", "evaluations"):
        assert np.array_equal(getattr(got, f)[[0, 4]], getattr(sub, f))


def test_rotation_profiles_skip_wide_ligands(docker):
    """gd_rotation_profiles is a warp-per-fragment kernel: a wide ligand in
    the staged batch is reported as skipped (status, message, no fragments)
    and the other ligands' profiles are unaffected."""
    pocket = W.config(1).pocket()
    c = pocket.mean(axis=0)
    small = _parts(W.config(1).ligands(range(3), c))
    ch = Lig(_zigzag(300), [(i, i + 1, i % 11 == 4) for i in range(299)], radius=0.8)
    wide = (ch.xyz + c - ch.xyz.mean(axis=0), ch.radii, ch.bonds, ch.rot)
    docker.set_pocket(pocket)
    mixed = docker.rotation_profiles(LigandBatch.from_parts([small[0], wide, small[1], small[2]]))
    alone = docker.rotation_profiles(LigandBatch.from_parts(small))
    assert mixed.status.tolist() == [0, 1, 0, 0]
    assert mixed.frag_offsets[2] == mixed.frag_offsets[1]  # no fragments for the wide ligand
    assert np.array_equal(mixed.scores, alone.scores) and np.array_equal(mixed.valid, alone.valid)
