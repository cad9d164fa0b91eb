"""Rotation-profile analysis on the CPU (reference analysis.hpp:17-217).

* The native host half (gd_detect_peaks, gd_tile_hit_probability) against
  the reference's own detect_peaks / tile_hit_probability (oracle/_ref),
  bit for bit, on the reference tests' hand cases (test_analysis.cpp:57-185)
  and on randomized profiles.
* The C oracle's rotation_profile restatement pinned to the reference's.
"""
import numpy as np
import pytest

from paper_1901_06363_b200 import GeoDockError
from paper_1901_06363_b200.analysis import detect_peaks, tile_hit_probability


def _oracle():
    from oracle import oracle_py
    return oracle_py


def _need_ref():
    O = _oracle()
    if not O.have_ref():
        pytest.skip("oracle/_ref not built")
    return O


def constant(value):
    return np.full(360, value, dtype=np.float64), np.ones(360, dtype=bool)


def as_tuple(st):
    return st.delta_overlap, st.best_peak_width, [(p.start_angle, p.width, p.height_ratio)
                                                 for p in st.peaks]


def test_single_rectangular_peak():
    s, v = constant(0.0)
    s[2] = s[3] = 1.0
    st = detect_peaks(s, v)
    assert as_tuple(st) == (1.0, 2, [(2, 2, 1.0)])


def test_flat_profile_has_no_peaks():
    st = detect_peaks(*constant(3.5))
    assert as_tuple(st) == (0.0, 0, [])


def test_runs_through_359_and_0_merge():
    s, v = constant(0.0)
    for a in (358, 359, 0, 1):
        s[a] = 1.0
    st = detect_peaks(s, v)
    assert [(p.start_angle, p.width) for p in st.peaks] == [(358, 4)]
    assert st.best_peak_width == 4


def test_all_invalid_is_an_error():
    with pytest.raises(GeoDockError, match="no feasible"):
        detect_peaks(np.zeros(360), np.zeros(360, dtype=bool))


def test_whole_circle_is_one_peak_and_mixed_validity():
    s = np.linspace(1.0, 2.0, 360)
    v = np.ones(360, dtype=bool)
    s[:] = 2.0
    s[100] = 1.0  # min at 100; everything else qualifies: one run through 0
    st = detect_peaks(s, v)
    assert [(p.start_angle, p.width) for p in st.peaks] == [(101, 359)]


def test_tile_hits_counts_model_monotone():
    hits = tile_hit_probability([68] * 10, [18, 90])
    assert (hits[0].probability, hits[1].probability, hits[0].eval_count) == (1.0, 0.0, 38.0)
    assert tile_hit_probability([68] * 10, []) == []
    table = tile_hit_probability([5, 20, 40, 68, 120, 200], [2, 6, 12, 18, 30, 60, 90, 180])
    assert all(b.probability <= a.probability for a, b in zip(table, table[1:]))
    with pytest.raises(GeoDockError):
        tile_hit_probability([], [18])


def _random_profiles(rng, count):
    """Profiles with plateaus, ties, wrap-around runs and invalid gaps."""
    for k in range(count):
        kind = k % 4
        s = rng.normal(size=360)
        if kind == 1:
            s = np.round(s, 1)  # many exact ties
        elif kind == 2:
            s = np.sin(np.deg2rad(np.arange(360) * rng.integers(1, 6)) + rng.uniform(0, 6.3))
        elif kind == 3:
            s = np.where(rng.random(360) < 0.5, 1.0, 0.25)
        v = rng.random(360) < rng.uniform(0.05, 1.0)
        yield s, v


def test_detect_peaks_matches_reference_randomized():
    O = _need_ref()
    rng = np.random.default_rng(99)
    n = 0
    for s, v in _random_profiles(rng, 400):
        want = O.ref_detect_peaks(s, v)
        if want is None:
            with pytest.raises(GeoDockError):
                detect_peaks(s, v)
            continue
        assert as_tuple(detect_peaks(s, v)) == want
        n += 1
    assert n > 300


def test_tile_hits_match_reference():
    O = _need_ref()
    rng = np.random.default_rng(5)
    widths = rng.integers(0, 361, size=1000)
    tiles = [1, 2, 3, 4, 5, 6, 8, 9, 10, 12, 15, 18, 20, 24, 30, 36, 40, 45, 60, 72, 90, 120, 180,
             360]
    prob, ev = O.ref_tile_hits(widths, tiles)
    got = tile_hit_probability(list(widths), tiles)
    assert [h.probability for h in got] == list(prob)
    assert [h.eval_count for h in got] == list(ev)


def test_oracle_profiles_pinned_to_reference():
    """The C restatement of rotation_profile vs the reference's own, bit for
    bit, on the reference generator's datasets (test_analysis.cpp:39-55)."""
    O = _need_ref()
    for count, seed in ((6, 1234), (8, 4096)):
        pocket, batch = O.ref_generate_synthetic(count, seed)
        a = O.rotation_profiles(batch, pocket, "oracle")
        b = O.rotation_profiles(batch, pocket, "ref", nthreads=O.threads())
        for x, y in zip(a, b):
            assert np.array_equal(x, y)
        assert len(a[0]) > 10


def test_oracle_profile_far_rigid_pair_valid_everywhere():
    """test_analysis.cpp:26-37: a two-atom fragment cannot bump."""
    from paper_1901_06363_b200 import LigandBatch
    O = _oracle()
    batch = LigandBatch.from_parts([(np.array([[0, 0, 0], [0, 0, 1.4], [1.2, 0, 1.4]], float),
                                     np.ones(3), np.array([[0, 1], [1, 2]]), np.array([1, 0]))])
    pocket = np.array([[0.0, 0.0, 1.0]])
    scores, valid, rel, offs, status = O.rotation_profiles(batch, pocket, "oracle")
    assert offs.tolist() == [0, 2] and valid.all()
    assert scores[1, 0] == O.overlap_score(batch.xyz, pocket)
