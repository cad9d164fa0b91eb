"""Full-size checks on BASELINE config 1 (10,000 ligands x 1 pocket).

At this size the reference itself still finishes in about a minute on the
box's host cores (oracle/_ref with its PocketIndex), so the whole workload
is compared bit for bit.  Size-independent properties are checked as well:
E7 ordering, E8 counters, seed-rank permutations, monotone refinement
(match_probes_shape never returns a worse score than its seed), final score
= overlap_score(final pose) re-scored by the independent scoring kernel,
and run-to-run determinism.
"""
import numpy as np
import pytest

from paper_1901_06363_b200 import workloads as W
from gd_test_helpers import assert_same_result

pytestmark = pytest.mark.gpu


def _oracle():
    from oracle import oracle_py
    return oracle_py


def test_config1_full_workload(docker):
    w = W.config(1)
    pocket = w.pocket()
    batch = w.ligands(range(w.n_ligands), pocket.mean(axis=0))
    knobs = w.knobs
    K = knobs.top_k
    docker.set_pocket(pocket)
    got = docker.dock(batch, knobs, keep_poses=True)

    n_orient = 744  # distinct Euler orientations at 30 degrees (E2)
    assert (got.status == 0).all() and (got.k_eff == K).all()
    # E8: poses scored = rigid orientations + the chains' evaluations.
    assert np.array_equal(got.poses_scored, n_orient + got.evaluations.sum(axis=1))
    # E7: (final score desc, seed rank asc); seed ranks are a permutation.
    f, r = got.final_score, got.seed_rank
    assert ((f[:, :-1] > f[:, 1:]) | ((f[:, :-1] == f[:, 1:]) & (r[:, :-1] < r[:, 1:]))).all()
    assert (np.sort(r, axis=1) == np.arange(K)).all()
    # E5 through the seeds: rigid score by seed rank is non-increasing.
    by_rank = np.take_along_axis(got.rigid_score, np.argsort(r, axis=1), axis=1)
    assert (by_rank[:, :-1] >= by_rank[:, 1:]).all()
    # match_probes_shape never ends below its starting score.
    assert (got.final_score >= got.rigid_score).all()
    # Final score == overlap_score(final pose), re-scored by the scoring
    # kernel (an independent code path) for every pose of 1,000 ligands.
    sizes = batch.sizes
    for n in np.unique(sizes[:1000]):
        ligs = [l for l in range(1000) if sizes[l] == n]
        poses = np.stack([got.pose(batch, l, e) for l in ligs for e in range(K)])
        want = got.final_score[ligs].reshape(-1)
        assert np.array_equal(docker.overlap_scores(poses), want)
    # Determinism (a second, differently pipelined run: resident path).
    docker.upload(batch)
    docker.dock_resident(knobs)
    from paper_1901_06363_b200 import DockResult
    again = docker.download(DockResult.empty(batch.n_ligands, K, int(batch.atom_offsets[-1]), False))
    assert_same_result(again, got, poses=False)

    # The reference on the whole workload (or the C oracle on a subset).
    O = _oracle()
    if O.have_ref():
        want = O.dock_batch(batch, pocket, knobs, nthreads=O.threads(), keep_poses=False, impl="ref")
        assert_same_result(got, want, poses=False, ctx="full c1 vs reference: ")
    else:
        sub = list(range(0, w.n_ligands, 97))
        want = O.dock_batch(batch.subset(sub), pocket, knobs, nthreads=O.threads())
        for i, l in enumerate(sub):
            assert np.array_equal(got.final_score[l], want.final_score[i])
            assert np.array_equal(got.orientation[l], want.orientation[i])
