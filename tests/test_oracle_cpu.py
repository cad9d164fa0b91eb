"""Pins the CPU oracle (oracle/gd_oracle.c) to the reference.

The reference's own known-answer tests (test_geometry.cpp, test_kernel.cpp)
restated against the oracle, plus the golden vectors in tests/golden/ that
the reference itself produced (tests/golden/make_golden.py).  CPU only.
"""
import math
from pathlib import Path

import numpy as np
import pytest

from gd_test_helpers import Lig, assert_same_result, bump_probe, chain, peak_rig
from paper_1901_06363_b200 import DockResult, Knobs, LigandBatch

GOLDEN = Path(__file__).resolve().parent / "golden"


@pytest.fixture(scope="module")
def O():
    from oracle import oracle_py
    return oracle_py


# --------------------------------------------------------------------------
# overlap_score (test_geometry.cpp:45-82)
# --------------------------------------------------------------------------
def test_overlap_score_hand_values(O):
    assert O.overlap_score([[0, 0, 0]], [[0, 0, 1]]) == 1.0
    assert O.overlap_score([[0, 0, 0], [0, 0, 3]], [[0, 0, 0]]) == 2.0 / (1e-12 + 9.0)
    assert O.overlap_score([[0, 0, 2]], [[0, 0, 1], [0, 0, 4]]) == 1.0


def test_overlap_score_decreases_with_distance(O):
    prev = O.overlap_score([[0, 0, 1]], [[0, 0, 0]])
    for r in np.arange(1.5, 10.0, 0.5):
        cur = O.overlap_score([[0, 0, r]], [[0, 0, 0]])
        assert cur < prev
        prev = cur


def test_overlap_score_rigid_transform_invariance(O):
    z = np.load(GOLDEN / "reference_kernel.npz")
    rng = np.random.default_rng(11)
    ao, xyz, pocket = z["d0_atom_offsets"], z["d0_xyz"], z["d0_pocket"]
    for l in range(5):
        pose = xyz[ao[l]:ao[l + 1]]
        axis = rng.uniform(-1, 1, 3)
        axis /= np.linalg.norm(axis)
        ang, t = 3 * rng.uniform(-1, 1), 5 * rng.uniform(-1, 1, 3)

        def apply(p):
            c, s = math.cos(ang), math.sin(ang)
            return p * c + np.cross(axis, p) * s + np.outer(p @ axis, axis) * (1 - c) + t

        ref = O.overlap_score(pose, pocket)
        assert O.overlap_score(apply(pose), apply(pocket)) == pytest.approx(ref, rel=1e-9)


# --------------------------------------------------------------------------
# rotate_fragment (test_geometry.cpp:84-170)
# --------------------------------------------------------------------------
def test_rotate_quarter_turns(O):
    lig = Lig([[0, 0, 0], [0, 0, 1], [1, 0, 1]], [(0, 1, True), (1, 2, False)])
    out, _ = O.rotate_fragment(*lig.args, lig.xyz, 1, 90.0)  # right fragment, axis 1->0 (-z)
    np.testing.assert_allclose(out[2], [0, -1, 1], atol=1e-12)
    assert np.array_equal(out[:2], lig.xyz[:2])
    lig2 = Lig([[1, 0, 0], [0, 0, 0], [0, 0, 1]], [(0, 1, False), (1, 2, True)])
    out2, _ = O.rotate_fragment(*lig2.args, lig2.xyz, 0, 90.0)  # left {0,1}, axis 1->2 (+z)
    np.testing.assert_allclose(out2[0], [0, 1, 0], atol=1e-12)


def test_rotate_identity_and_full_turn(O):
    z = np.load(GOLDEN / "reference_kernel.npz")
    for d in range(2):
        b = _batch(z, f"d{d}_")
        for l in range(b.n_ligands):
            x, r, bd, ro = b.ligand(l)
            for f in range(0, 2 * int(ro.sum()), 2):
                zero, _ = O.rotate_fragment(x, r, bd, ro, x, f, 0.0)
                assert np.array_equal(zero, x)
                full, _ = O.rotate_fragment(x, r, bd, ro, x, f, 360.0)
                np.testing.assert_allclose(full, x, atol=1e-9)


def test_rotate_rigid_and_invertible(O):
    z = np.load(GOLDEN / "reference_kernel.npz")
    b = _batch(z, "d1_")
    rng = np.random.default_rng(5)
    for l in range(b.n_ligands):
        x, r, bd, ro = b.ligand(l)
        for f in range(0, 2 * int(ro.sum()), 2):
            th = rng.uniform(1, 359)
            rot, _ = O.rotate_fragment(x, r, bd, ro, x, f, th)
            back, _ = O.rotate_fragment(x, r, bd, ro, rot, f, -th)
            np.testing.assert_allclose(back, x, atol=1e-9)
            moved = np.any(rot != x, axis=1)
            idx = np.where(moved)[0]
            for i in idx:
                for j in idx:
                    assert abs(np.linalg.norm(rot[i] - rot[j]) - np.linalg.norm(x[i] - x[j])) < 1e-9


def test_rotate_degenerate_axis(O):
    lig = chain([[0, 0, 0], [1.5, 0, 0], [3, 0, 0]])
    pose = lig.xyz.copy()
    pose[1] = pose[0]
    with pytest.raises(RuntimeError):
        O.rotate_fragment(*lig.args, pose, 0, 10.0)
    if O.have_ref():
        with pytest.raises(RuntimeError, match="degenerate"):
            O.rotate_fragment(*lig.args, pose, 0, 10.0, impl="ref")


# --------------------------------------------------------------------------
# check_bumps (test_geometry.cpp:191-234)
# --------------------------------------------------------------------------
def test_bump_rule(O):
    lig = bump_probe(0.1, 1.5)
    _, feas = O.rotate_fragment(*lig.args, lig.xyz, 0, 0.0)
    assert not feas
    lig = bump_probe(2.5, 1.5)
    _, feas = O.rotate_fragment(*lig.args, lig.xyz, 0, 0.0)
    assert feas
    fold = Lig([[0, 0, 0], [1.5, 0, 0], [1.5, 1.5, 0], [0.1, 0.1, 0]],
               [(0, 1, False), (1, 2, True), (2, 3, False)], 1.5)
    _, feas = O.rotate_fragment(*fold.args, fold.xyz, 0, 0.0)
    assert feas  # graph distance 3: excluded by the 1-4 rule


def _bfs(n, bonds):
    adj = [[] for _ in range(n)]
    for a, b in bonds:
        adj[a].append(b)
        adj[b].append(a)
    dist = np.full((n, n), -1)
    for s in range(n):
        dist[s, s] = 0
        q = [s]
        for at in q:
            for nb in adj[at]:
                if dist[s, nb] < 0:
                    dist[s, nb] = dist[s, at] + 1
                    q.append(nb)
    return dist


def test_bumps_match_all_pairs_oracle(O):
    """bump_oracle (oracles.hpp:51-81) restated in numpy, every 23 degrees."""
    z = np.load(GOLDEN / "reference_kernel.npz")
    b = _batch(z, "d4_")  # small_dataset(10, 2024)
    bumped = feasible = 0
    for l in range(b.n_ligands):
        x, r, bd, ro = b.ligand(l)
        dist = _bfs(len(x), bd)
        for f in range(0, 2 * int(ro.sum()), 2):
            for ang in range(0, 360, 23):
                cand, fast = O.rotate_fragment(x, r, bd, ro, x, f, float(ang))
                moved = _left_members(len(x), bd, ro, f)
                ok = True
                for i in np.where(moved)[0]:
                    for j in np.where(~moved)[0]:
                        if dist[i, j] >= 4 and np.linalg.norm(cand[i] - cand[j]) < 0.8 * (r[i] + r[j]):
                            ok = False
                assert fast == ok
                bumped += not ok
                feasible += ok
    assert bumped > 0 and feasible > 0


def _left_members(n, bonds, rot, f):
    rots = sorted((min(a, b), max(a, b), k) for k, (a, b) in enumerate(bonds) if rot[k])
    lo, hi, k = rots[f // 2]
    adj = [[] for _ in range(n)]
    for kk, (a, b) in enumerate(bonds):
        if kk != k:
            adj[a].append(b)
            adj[b].append(a)
    seen = np.zeros(n, bool)
    seen[lo] = True
    q = [lo]
    for at in q:
        for nb in adj[at]:
            if not seen[nb]:
                seen[nb] = True
                q.append(nb)
    return seen if f % 2 == 0 else ~seen


# --------------------------------------------------------------------------
# kernel.hpp searches (test_kernel.cpp:35-263)
# --------------------------------------------------------------------------
def test_optimal_tile_size(O):
    tile = O.oracle().gdo_optimal_tile_size
    assert tile(1) == 18 and tile(4) == 36 and tile(360) == 360
    z = np.load(GOLDEN / "reference_kernel.npz")
    assert [tile(s) for s in range(1, 361)] == z["tile_sizes"].tolist()


def test_flat_search_counts_and_peak(O):
    lig, pocket = peak_rig()
    a, s, ev, ck, pose = O.optimize_fragment(*lig.args, pocket, 1, 360)
    assert (a, ev, ck) == (0, 1, 1) and np.array_equal(pose, lig.xyz)
    _, _, ev, ck, _ = O.optimize_fragment(*lig.args, pocket, 1, 90)
    assert ck == 4 and ev <= 4
    a, *_ = O.optimize_fragment(*lig.args, pocket, 1, 30)
    assert a == 90


def test_refined_search(O):
    lig, pocket = peak_rig()
    _, s, ev, ck, _ = O.optimize_fragment(*lig.args, pocket, 1, 1, refined=True)
    assert ev <= 38 and s >= O.overlap_score(lig.xyz, pocket)
    axial = Lig([[0, 0, 0], [0, 0, 1]], [(0, 1, True)])
    a, *_ = O.optimize_fragment(*axial.args, np.array([[0.5, 0, 1]]), 1, 1, refined=True)
    assert a == 9  # constant profile: centre of tile [0, 18)


def test_refined_captures_wide_peak(O):
    lig = Lig([[0, 0, 0], [0, 0, 1], [1, 0, 1]], [(0, 1, True), (1, 2, False)])
    probe99, _ = O.rotate_fragment(*lig.args, lig.xyz, 1, 99.0)
    pocket = np.array([[0, 0, 0], [0, 0, 1.585], probe99[2]])
    fa, fs, *_, fpose = O.optimize_fragment(*lig.args, pocket, 1, 1)
    ra, rs, *_, rpose = O.optimize_fragment(*lig.args, pocket, 1, 1, refined=True)
    assert fa == 99 and ra == 99 and fs == rs and np.array_equal(fpose, rpose)


def test_match_probes_shape_counts(O):
    lig, pocket = peak_rig()
    s, ev, ck, _ = O.match_probes_shape(*lig.args, pocket, Knobs(1, 45, 0.0, 3, False))
    assert ck == 1 + 3 * 2 * 360 and ev <= ck
    _, ev, _, _ = O.match_probes_shape(*lig.args, pocket, Knobs(1, 45, 0.0, 1, True))
    assert ev <= 1 + 2 * 38
    _, _, ck, _ = O.match_probes_shape(*lig.args, pocket, Knobs(1, 90, 1.0, 1, False))
    assert ck == 1 + 2 * 4
    rigid = Lig([[0, 0, 0], [0, 0, 1.5]], [(0, 1, False)])
    s, ev, _, pose = O.match_probes_shape(*rigid.args, np.array([[0, 0, 1.0]]), Knobs())
    assert ev == 1 and s == O.overlap_score(rigid.xyz, [[0, 0, 1.0]])
    assert np.array_equal(pose, rigid.xyz)


def test_match_probes_shape_committed_and_monotone(O):
    z = np.load(GOLDEN / "reference_kernel.npz")
    b, pocket = _batch(z, "d0_"), z["d0_pocket"]  # small_dataset(10, 321)
    for l in range(b.n_ligands):
        x, r, bd, ro = b.ligand(l)
        a = O.match_probes_shape(x, r, bd, ro, pocket, Knobs(2, 90, 0.3, 2, True))
        c = O.match_probes_shape(x, r, bd, ro, pocket, Knobs(2, 90, 0.3, 2, True))
        assert a[0] == c[0] and np.array_equal(a[3], c[3]) and a[1] == c[1]
        assert a[0] == O.overlap_score(a[3], pocket)
        assert a[0] >= O.overlap_score(x, pocket)
    b, pocket = _batch(z, "d1_"), z["d1_pocket"]  # small_dataset(5, 555)
    for l in range(b.n_ligands):
        x, r, bd, ro = b.ligand(l)
        prev = None
        for step in (1, 2, 3, 5, 10):
            ev = O.match_probes_shape(x, r, bd, ro, pocket, Knobs(step, 90, 0.0, 1, False))[1]
            assert prev is None or ev <= prev
            prev = ev
        once = O.match_probes_shape(x, r, bd, ro, pocket, Knobs(5, 90, 0.0, 1, False))[2]
        thrice = O.match_probes_shape(x, r, bd, ro, pocket, Knobs(5, 90, 0.0, 3, False))[2]
        assert thrice - 1 == 3 * (once - 1)


def test_algorithm1_equivalence(O):
    """algorithm1_dock (oracles.hpp:26-47), restated, vs match_probes_shape{1,45,0,1}."""
    z = np.load(GOLDEN / "reference_kernel.npz")
    b, pocket = _batch(z, "d2_"), z["d2_pocket"]  # small_dataset(12, 4242)
    for l in range(6):
        x, r, bd, ro = b.ligand(l)
        pose = x.copy()
        final = O.overlap_score(pose, pocket)
        for f in range(2 * int(ro.sum())):
            best_a, best = 0, O.overlap_score(pose, pocket)
            for ang in range(1, 360):
                cand, feas = O.rotate_fragment(x, r, bd, ro, pose, f, float(ang))
                if not feas:
                    continue
                s = O.overlap_score(cand, pocket)
                if s > best:
                    best, best_a = s, ang
            if best_a:
                pose, _ = O.rotate_fragment(x, r, bd, ro, pose, f, float(best_a))
            final = best
        assert O.match_probes_shape(x, r, bd, ro, pocket, Knobs(1, 45, 0.0, 1, False))[0] == final


# --------------------------------------------------------------------------
# Golden vectors produced by the reference itself
# --------------------------------------------------------------------------
def _batch(z, p):
    return LigandBatch(z[p + "atom_offsets"], z[p + "xyz"], z[p + "radii"], z[p + "bond_offsets"],
                       z[p + "bonds"], z[p + "rotatable"])


def test_oracle_matches_reference_match_probes_shape_golden(O):
    z = np.load(GOLDEN / "reference_kernel.npz")
    knobs = [Knobs(int(k[0]), int(k[1]), float(k[2]), int(k[3]), bool(k[4])) for k in z["knobs"]]
    for d in range(6):
        b, pocket = _batch(z, f"d{d}_"), z[f"d{d}_pocket"]
        for ki, kn in enumerate(knobs):
            poses = []
            for l in range(b.n_ligands):
                x, r, bd, ro = b.ligand(l)
                s, ev, ck, pose = O.match_probes_shape(x, r, bd, ro, pocket, kn)
                assert s == z[f"d{d}_k{ki}_score"][l], (d, ki, l)
                assert ev == z[f"d{d}_k{ki}_evals"][l] and ck == z[f"d{d}_k{ki}_checks"][l]
                poses.append(pose)
            assert np.array_equal(np.concatenate(poses), z[f"d{d}_k{ki}_pose"])


@pytest.mark.parametrize("name", ["c0", "c1", "c2"])
def test_oracle_matches_reference_baseline_golden(O, name):
    z = np.load(GOLDEN / "baseline_configs.npz")
    b, pocket = _batch(z, f"{name}_"), z[f"{name}_pocket"]
    k = z[f"{name}_knobs"]
    knobs = Knobs(int(k[0]), int(k[1]), float(k[2]), int(k[3]), bool(k[4]), int(k[5]), int(k[6]))
    got = O.dock_batch(b, pocket, knobs, nthreads=O.threads())
    want = DockResult(*(z[f"{name}_{f}"] for f in (
        "orientation", "seed_rank", "rigid_score", "final_score", "evaluations",
        "feasibility_checks", "k_eff", "poses_scored", "status", "final_pose")))
    assert_same_result(got, want, ctx=name + ": ")


def test_orientation_grid_counts(O):
    """E2 de-duplication: distinct Euler-grid rotations (SURVEY.md §8(a) E2 probe counts)."""
    for step, n in [(45, 208), (30, 744), (20, 2916), (15, 6384), (10, 22104)]:
        idx, R = O.orientations(step)
        assert len(idx) == n and idx[0] == 0
        assert np.array_equal(R[0], np.eye(3))
        np.testing.assert_allclose(R @ R.transpose(0, 2, 1), np.broadcast_to(np.eye(3), R.shape),
                                   atol=1e-12)
