"""Pins of the oracle's full-covariance CEM (DESIGN reading L42):
Alg. 1 UpdateCov with a full C, sampling theta2 = mu' + L z with the same
normative noise z.  Each check reduces to a library routine (numpy Cholesky, cov,
matvec), to the already-pinned diagonal sampler / CEM update, or to statistics.
"""
import numpy as np
import pytest

from paper_2403_11383_b200 import workloads as W


def _spd(D, seed):
    rng = np.random.default_rng(seed)
    A = rng.normal(size=(D, D))
    return A @ A.T / D + np.diag(rng.uniform(0.5, 2.0, D))


@pytest.mark.parametrize("D", [1, 2, 24, 48, 96])
def test_cholesky_is_the_library_factor(orc, D):
    Cm = _spd(D, D)
    rc, Lm = orc.cholesky(Cm)
    assert rc == 0
    np.testing.assert_allclose(Lm, np.linalg.cholesky(Cm), rtol=1e-12, atol=1e-12)
    assert np.all(np.triu(Lm, 1) == 0)


def test_cholesky_rejects_indefinite(orc):
    Cm = np.array([[1.0, 2.0], [2.0, 1.0]])
    assert orc.cholesky(Cm)[0] == -1


def test_diagonal_factor_reproduces_the_diagonal_sampler(orc):
    cfg = W.base_config(n_samples=64, mode="cem", n_elite=8, gait_adapt=1)
    st = W.initial_distribution(cfg)
    mu_s = orc.warm_shift(cfg, st["mean"])
    Lm = np.diag(np.sqrt(st["var"]))
    for k in range(0, 30):
        a = orc.sample(cfg, mu_s, st["var"], 1, 5, 2, k)
        b = orc.sample_full(cfg, mu_s, Lm, 1, 5, 2, k)
        np.testing.assert_array_equal(a[0], b[0])
        np.testing.assert_array_equal(a[1], b[1])
        assert a[2] == b[2]


def test_full_factor_sample_is_mu_plus_L_z(orc):
    cfg = W.base_config(n_samples=64, mode="cem", n_elite=8)
    st = W.initial_distribution(cfg)
    mu_s = orc.warm_shift(cfg, st["mean"])
    Lm = np.linalg.cholesky(_spd(48, 3) * 20.0)
    for k in (1, 2, 17, 63):
        th, z, _ = orc.sample_full(cfg, mu_s, Lm, 0, 0, 0, k)
        _, z_diag, _ = orc.sample(cfg, mu_s, st["var"], 0, 0, 0, k)
        np.testing.assert_array_equal(z, z_diag)                       # same normative noise
        np.testing.assert_allclose(th, mu_s + Lm @ z.astype(np.float64), rtol=1e-13, atol=1e-10)
    th0, _, _ = orc.sample_full(cfg, mu_s, Lm, 0, 0, 0, 0)            # elite preservation
    np.testing.assert_array_equal(th0, mu_s)


def test_full_factor_sample_covariance(orc):
    cfg = W.base_config(n_samples=64, knots=2, elite_preserve=0)         # D = 24
    D = 24
    mu = np.zeros(D)
    Cm = _spd(D, 9) * 10.0
    Lm = np.linalg.cholesky(Cm)
    X = np.array([orc.sample_full(cfg, mu, Lm, 0, 0, 0, k)[0] for k in range(20000)])
    Ce = np.cov(X.T, bias=True)
    err = np.abs(Ce - Cm) / np.sqrt(np.outer(np.diag(Cm), np.diag(Cm)))   # correlation units
    assert err.max() < 0.05


def test_update_full_with_all_elites_is_the_population_covariance(orc):
    rng = np.random.default_rng(5)
    K, D = 300, 12
    J = rng.uniform(0, 10, K)
    th = rng.normal(size=(K, D)) @ rng.normal(size=(D, D))
    floor = np.full(D, 0.01)
    rc, mu, Cn, Ln, e, dg = orc.cem_update_full(J, th, K, floor)
    assert rc == 0
    np.testing.assert_allclose(mu, th.mean(0), rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(Cn, np.cov(th.T, bias=True) + np.diag(floor), rtol=1e-10, atol=1e-12)
    np.testing.assert_allclose(Ln, np.linalg.cholesky(Cn), rtol=1e-10, atol=1e-12)


def test_update_full_diagonal_matches_the_pinned_diagonal_update(orc):
    """diag(C_new) - floor = the elite variance of the (pinned) diagonal update; same mean, same elites."""
    rng = np.random.default_rng(6)
    K, D, Ke = 500, 48, 60
    J = rng.uniform(0, 10, K)
    J[[3, 9]] = np.inf
    th = rng.normal(size=(K, D)) * 5 + 3
    floor = np.full(D, 1e-6)
    rc, mu, Cn, Ln, e, dg = orc.cem_update_full(J, th, Ke, floor)
    rc2, mu2, var2, e2, dg2 = orc.cem_update(J, th, Ke, floor, 1, np.ones(D))
    assert rc == rc2 == 0
    np.testing.assert_array_equal(e, e2)
    np.testing.assert_array_equal(mu, mu2)
    np.testing.assert_allclose(np.diag(Cn) - floor, var2, rtol=1e-12)


def test_step_first_iteration_matches_diagonal_cem(orc):
    """From C = diag(sigma^2) the first full-covariance iteration draws the same samples and
    elites as the diagonal CEM, hence the same new mean."""
    cfg, inputs = W.config3("cem", K=400)
    cfg = dict(cfg, n_elite=60)
    full = dict(cfg, full_cov=1)
    a = orc.step(cfg, 0, inputs[0], W.initial_distribution(cfg))
    st = W.initial_distribution(full)
    b = orc.step(full, 0, inputs[0], st)
    np.testing.assert_array_equal(a.theta, b.theta)
    np.testing.assert_array_equal(a.elite, b.elite)
    np.testing.assert_array_equal(a.mean, b.mean)
    Lm = st["chol"]
    np.testing.assert_allclose(np.diag(Lm @ Lm.T), b.var, rtol=1e-12)
    assert np.all(np.triu(Lm, 1) == 0) and np.any(np.abs(np.tril(Lm, -1)) > 0)
