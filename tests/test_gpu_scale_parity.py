"""Parity at every BASELINE configuration's own scale (north_star: "for every
config, the selected pose indices and ordering of each ligand's top-K match
the CPU oracle exactly").

The checker is the reference itself: its headers compiled from
/root/reference into oracle/_ref (PocketIndex, fp64, 16 host threads),
driven through oracle/ref_harness.cpp's rigid sweep + top-K + restart
chains of the reference match_probes_shape (kernel.hpp:205-248).  Where
oracle/_ref is absent the plain-C restatement stands in.

* c2: 200 ligands at rigid 10, fragment 10, 3 restarts, K = 100 (22,104
  orientations through the rank-merge top-K, 35-candidate fragment
  searches in 6-batches).
* c3: all 16 pockets (1 A lattice, semi-axes U(5,12) A, roughness mask)
  x 64 ligands each; the smallest, largest and roughest pockets are named
  in the test ids.
* c4: every one of the 180 knob points (rigid {10,15,20,30,45} x fragment
  {10,20,30,60} x restarts {1,2,3} x K {10,30,100}) on 4 ligands, the
  points spread over c4's four pockets.

Bar: bit-exact top-K orientation indices, order, seed ranks, rigid and
final scores, evaluation and feasibility-check counters and final poses.
"""
import itertools

import numpy as np
import pytest

from paper_1901_06363_b200 import Knobs, workloads as W
from gd_test_helpers import assert_same_result

pytestmark = pytest.mark.gpu


def _cpu(batch, pocket, knobs, poses=True):
    from oracle import oracle_py as O
    impl = "ref" if O.have_ref() else "oracle"
    return O.dock_batch(batch, pocket, knobs, nthreads=O.threads(), keep_poses=poses, impl=impl)


def test_config2_200_ligands(docker):
    w = W.config(2)
    pocket = w.pocket()
    batch = w.ligands(range(200))
    docker.set_pocket(pocket)
    got = docker.dock(batch, w.knobs, keep_poses=True)
    assert (got.status == 0).all() and (got.k_eff == 100).all()
    want = _cpu(batch, pocket, w.knobs)
    assert_same_result(got, want, ctx="c2 x200: ")


def _c3_pockets():
    w = W.config(3)
    pockets = [W.pocket_of(w, p) for p in range(16)]
    full = [len(W.synth_pocket_unrough(w, p)) for p in range(16)]
    rough = [1.0 - len(pk) / f for pk, f in zip(pockets, full)]
    sizes = [len(pk) for pk in pockets]
    tags = {}
    tags[int(np.argmin(sizes))] = "smallest"
    tags[int(np.argmax(sizes))] = "largest"
    tags[int(np.argmax(rough))] = tags.get(int(np.argmax(rough)), "") + "roughest"
    ids = [f"p{p}-P{sizes[p]}-rough{100 * rough[p]:.0f}pct" + (f"-{tags[p]}" if p in tags else "")
           for p in range(16)]
    return w, pockets, ids


_C3 = None


def _c3():
    global _C3
    if _C3 is None:
        _C3 = _c3_pockets()
    return _C3


@pytest.mark.parametrize("p", range(16), ids=lambda p: f"pocket{p}")
def test_config3_every_pocket(docker, p):
    w, pockets, ids = _c3()
    pocket = pockets[p]
    batch = w.ligands(range(64 * p, 64 * p + 64), pocket.mean(axis=0))
    docker.set_pocket(pocket)
    got = docker.dock(batch, w.knobs, keep_poses=True)
    assert (got.status == 0).all()
    want = _cpu(batch, pocket, w.knobs)
    assert_same_result(got, want, ctx=f"c3 {ids[p]}: ")


C4_GRID = list(itertools.product([10, 15, 20, 30, 45], [10, 20, 30, 60], [1, 2, 3], [10, 30, 100]))


def test_config4_grid_is_complete():
    assert len(C4_GRID) == 180


@pytest.mark.parametrize("point", range(len(C4_GRID)),
                         ids=lambda i: "r{}-f{}-x{}-k{}".format(*C4_GRID[i]))
def test_config4_every_knob_point(docker, point):
    w = W.config(4)
    g = C4_GRID[point]
    pocket = W.pocket_of(w, point % 4)
    batch = w.ligands(range(4 * point, 4 * point + 4), pocket.mean(axis=0))
    knobs = Knobs.baseline(*g)
    docker.set_pocket(pocket)
    got = docker.dock(batch, knobs, keep_poses=True)
    assert (got.status == 0).all()
    want = _cpu(batch, pocket, knobs)
    assert_same_result(got, want, ctx=f"c4 {g}: ")


def test_hollow_shell_pocket_overflow_voxels(docker):
    """A hollow spherical shell: near the centre no surface point dominates
    another, so interior voxels keep more than 1,024 candidates.  Those
    voxels scan the whole pocket (held once at the head of the list array)
    instead of listing it per voxel; minima stay exact and the index stays
    small."""
    m = 1500  # Fibonacci sphere of radius 8 A: equidistant from the centre
    k = np.arange(m) + 0.5
    phi, th = np.arccos(1 - 2 * k / m), np.pi * (1 + 5 ** 0.5) * k
    shell = 8.0 * np.stack([np.cos(th) * np.sin(phi), np.sin(th) * np.sin(phi), np.cos(phi)], 1)
    docker.set_pocket(shell)
    info = docker.pocket_info()
    # Without the shared head every overflow voxel would list the whole shell.
    assert info["max_candidates"] == len(shell)
    rng = np.random.default_rng(7)
    poses = rng.uniform(-13.0, 13.0, size=(512, 24, 3))
    poses[:128] *= 0.05  # deep inside: the overflow voxels
    a = docker.overlap_scores(poses)
    b = docker.overlap_scores(poses, brute=True)
    assert np.array_equal(a, b)
    from oracle import oracle_py as O
    want = np.array([O.overlap_score(q, shell) for q in poses[:64]])
    assert np.array_equal(a[:64], want)


def test_fixed_point_replay_many_restarts(docker):
    """Chains with several restarts stop searching once every fragment has
    kept angle 0 in a row and replay the remaining steps' counts
    (flex_chain_kernel, kReplay).  Eight restarts make most steps replays;
    the zig-zag ligand has more than 32 fragments, so its chains run every
    step; scores, poses and both CandidateEvaluator counters must still
    equal the reference's, which searches every step."""
    from paper_1901_06363_b200 import LigandBatch
    from gd_test_helpers import Lig
    from test_gpu_prep import _zigzag
    w = W.config(1)
    pocket = w.pocket()
    c = pocket.mean(axis=0)
    base = w.ligands(range(12))
    long = Lig(_zigzag(40), [(i, i + 1, True) for i in range(39)], radius=0.9)  # 37 rotamers
    parts = [(base.xyz[base.atom_offsets[l]:base.atom_offsets[l + 1]],
              base.radii[base.atom_offsets[l]:base.atom_offsets[l + 1]],
              base.bonds[base.bond_offsets[l]:base.bond_offsets[l + 1]],
              base.rotatable[base.bond_offsets[l]:base.bond_offsets[l + 1]]) for l in range(12)]
    parts.append((long.xyz + c - long.xyz.mean(axis=0), long.radii, long.bonds, long.rot))
    batch = LigandBatch.from_parts(parts)
    docker.set_pocket(pocket)
    for knobs in (Knobs.baseline(45, 30, 8, 6), Knobs(20, 60, 0.3, 5, True, 45, 4)):
        got = docker.dock(batch, knobs, keep_poses=True)
        assert (got.status == 0).all()
        want = _cpu(batch, pocket, knobs)
        assert_same_result(got, want, ctx=f"replay {knobs}: ")
