"""The planner's cost-model fit (reference perf_model.hpp:57-105) on the CPU.

The reference solves the OLS with Eigen (absent here), so gd_fit_cost_model
is pinned by the reference tests' own cases (test_perf_model.cpp:41-132:
exact recovery, pure noise, interpolation, rejections) and by an
independent solver, numpy's lstsq, on well-conditioned random systems.
"""
import numpy as np
import pytest

from paper_1901_06363_b200.native import GeoDockError, fit_cost_model


def features_of(rng, n):
    return np.stack([rng.uniform(20, 200, n).astype(int).astype(float), rng.uniform(5, 40, n),
                     rng.uniform(2, 12, n)], axis=1)


def design(f):
    pp, la, lr = f[:, 0], f[:, 1], f[:, 2]
    return np.stack([pp, la, lr, pp * la, pp * lr, la * lr, pp * la * lr, np.ones(len(f))], axis=1)


def test_recovers_exact_coefficients_from_noiseless_data():
    rng = np.random.default_rng(1)
    truth = np.array([2e-5, 1e-4, 3e-4, 4e-7, 5e-7, 6e-6, 1e-8])
    f = features_of(rng, 40)
    t = design(f)[:, :7] @ truth + 0.01
    coef, icpt, r2 = fit_cost_model(f, t)
    np.testing.assert_allclose(coef, truth, rtol=1e-6)
    assert icpt == pytest.approx(0.01, rel=1e-6)
    assert r2 > 0.999999


def test_pure_noise_explains_nothing():
    rng = np.random.default_rng(2)
    f = features_of(rng, 2000)
    t = rng.uniform(0.5, 1.5, 2000)
    _, _, r2 = fit_cost_model(f, t)
    assert abs(r2) < 0.05


def test_interpolates_nine_general_position_observations():
    rng = np.random.default_rng(3)
    f = features_of(rng, 9)
    truth = rng.uniform(1e-8, 1e-5, 7)
    t = design(f)[:, :7] @ truth + 0.05
    coef, icpt, r2 = fit_cost_model(f, t)
    pred = design(f) @ np.append(coef, icpt)
    np.testing.assert_allclose(pred, t, rtol=1e-6)
    assert r2 == pytest.approx(1.0, abs=1e-9)


def test_matches_numpy_lstsq_on_well_conditioned_systems():
    rng = np.random.default_rng(4)
    for trial in range(20):
        n = int(rng.integers(12, 200))
        f = features_of(rng, n)
        t = rng.uniform(1e-3, 1.0, n)
        coef, icpt, r2 = fit_cost_model(f, t)
        X = design(f)
        want, *_ = np.linalg.lstsq(X, t, rcond=None)
        got = np.append(coef, icpt)
        sse_got = float(np.sum((t - X @ got) ** 2))
        sse_want = float(np.sum((t - X @ want) ** 2))
        assert sse_got == pytest.approx(sse_want, rel=1e-9, abs=1e-12)
        np.testing.assert_allclose(X @ got, X @ want, rtol=1e-7, atol=1e-10)
        sst = float(np.sum((t - t.mean()) ** 2))
        assert r2 == pytest.approx(1 - (sse_want / sst) * (n - 1) / (n - 8), rel=1e-9, abs=1e-12)


def test_rejects_too_few_and_rank_deficient():
    rng = np.random.default_rng(5)
    with pytest.raises(GeoDockError, match="at least 9 observations, got 8"):
        fit_cost_model(features_of(rng, 8), np.ones(8))
    la = rng.uniform(5, 40, 12)
    f = np.stack([np.full(12, 100.0), la, np.full(12, 4.0)], axis=1)
    with pytest.raises(GeoDockError, match="rank-deficient design matrix; collinear columns"):
        fit_cost_model(f, 0.5 + 0.001 * rng.uniform(5, 40, 12))
    with pytest.raises(GeoDockError, match="non-positive observation time"):
        fit_cost_model(features_of(rng, 10), np.r_[np.ones(9), 0.0])
