"""Pins for the distribution updates: MPPI (Alg. 4; O13) against
the worked weights, limits and a 50-digit brute force; CEM / Naive elite
selection (Alg. 1, 3; O14) against numpy's stable sort."""
import json
import math
import os
from decimal import Decimal, getcontext

import numpy as np
import pytest

GOLD = os.path.join(os.path.dirname(__file__), "golden")
PV = json.load(open(os.path.join(GOLD, "paper_values.json")))


def test_mppi_worked_two_costs(orc):
    g = PV["mppi_two_costs"]
    th = np.array([[1.0, 0.0], [0.0, 1.0]])
    rc, mu, dg = orc.mppi(g["J"], th, g["lambda"])
    assert rc == 0
    np.testing.assert_allclose(mu, g["w"], atol=1e-15)
    assert dg.j_min == 1.0 and dg.argmin == 0
    assert dg.omega == pytest.approx(1 + math.exp(-1))


def test_mppi_limits(orc):
    rng = np.random.default_rng(13)
    th = rng.normal(size=(40, 6))
    # all costs equal -> arithmetic mean
    rc, mu, _ = orc.mppi(np.full(40, 3.25), th, 1.0)
    np.testing.assert_allclose(mu, th.mean(0), atol=1e-14)
    # K = 1 -> that sample
    _, mu, _ = orc.mppi([7.0], th[:1], 1.0)
    np.testing.assert_allclose(mu, th[0], atol=0)
    # lambda -> 0 -> argmin sample (north star)
    J = rng.uniform(1, 2, 40)
    _, mu, dg = orc.mppi(J, th, 1e-6)
    np.testing.assert_allclose(mu, th[np.argmin(J)], atol=1e-14)
    # shift invariance
    _, mu1, _ = orc.mppi(J, th, 0.7)
    _, mu2, _ = orc.mppi(J + 123.0, th, 0.7)
    np.testing.assert_allclose(mu1, mu2, atol=1e-12)


def test_mppi_brute_force_50_digits(orc):
    getcontext().prec = 50
    rng = np.random.default_rng(14)
    K, D = 64, 48
    J = rng.uniform(0.5, 6.0, K)
    J[5] = math.inf                                # a diverged sample gets weight 0
    th = rng.normal(size=(K, D)) * 10
    rc, mu, dg = orc.mppi(J, th, 1.0)
    beta = Decimal(min(J))
    w = [Decimal(0) if not math.isfinite(j) else (-(Decimal(j) - beta)).exp() for j in J]
    Om = sum(w)
    for d in range(D):
        want = sum(wk * Decimal(th[k, d]) for k, wk in enumerate(w)) / Om
        assert abs(mu[d] - float(want)) < 1e-12 * max(1.0, abs(float(want)))
    assert dg.n_diverged == 1
    assert dg.ess == pytest.approx(float(Om * Om / sum(x * x for x in w)), rel=1e-12)


def test_mppi_all_diverged(orc):
    rc, mu, dg = orc.mppi([math.inf] * 4, np.ones((4, 3)), 1.0)
    assert rc == 1 and dg.n_diverged == 4


def test_naive_worked(orc):
    g = PV["naive_two_costs"]
    th = np.array([[1.0, 2.0], [3.0, 4.0]])
    rc, mu, var, e, dg = orc.cem_update(g["J"], th, 1, [0, 0], 0, [9.0, 9.0])
    assert e[0] == g["best"]
    np.testing.assert_array_equal(mu, th[g["best"]])
    np.testing.assert_array_equal(var, [9.0, 9.0])            # covariance unchanged


@pytest.mark.parametrize("K,Ke", [(64, 1), (64, 7), (64, 64), (1000, 100), (777, 300)])
def test_cem_select_equals_stable_sort(orc, K, Ke):
    rng = np.random.default_rng(K + Ke)
    J = rng.integers(0, 20, K).astype(np.float64)  # many exact ties
    J[rng.integers(0, K, 5)] = math.inf
    J[rng.integers(0, K, 3)] = math.nan
    e = orc.cem_select(J, Ke)
    key = np.where(np.isnan(J), math.inf, J)
    want = np.argsort(key, kind="stable")[:Ke]
    np.testing.assert_array_equal(e, want)


def test_cem_moments(orc):
    rng = np.random.default_rng(15)
    K, D, Ke = 200, 12, 30
    J = rng.uniform(0, 1, K)
    th = rng.normal(size=(K, D)) * 5
    floor = np.full(D, 0.5)
    rc, mu, var, e, dg = orc.cem_update(J, th, Ke, floor, 1, np.ones(D))
    sel = np.argsort(J, kind="stable")[:Ke]
    np.testing.assert_allclose(mu, th[sel].mean(0), atol=1e-12)
    np.testing.assert_allclose(var, np.maximum(th[sel].var(0), floor), atol=1e-12)
    # K_e = K: population moments
    rc, mu, var, e, dg = orc.cem_update(J, th, K, np.zeros(D), 1, np.ones(D))
    np.testing.assert_allclose(mu, th.mean(0), atol=1e-12)
    np.testing.assert_allclose(var, th.var(0), atol=1e-12)


@pytest.mark.parametrize("K,Ke,n_inf", [(50, 20, 40), (64, 64, 10), (200, 30, 185), (10, 10, 9)])
def test_cem_fewer_finite_than_elites(orc, K, Ke, n_inf):
    """Alg. 1 refits on the elite set; L17: a diverged rollout (J = +inf,
    L26) never enters the moments.  With fewer finite costs than K_e the elite list
    still holds K_e indices in (J, k) order (+inf last), and mean / variance are the
    population moments of the finite samples only (numpy on that subset)."""
    rng = np.random.default_rng(K * 7 + n_inf)
    D = 9
    J = rng.uniform(0, 5, K)
    J[rng.permutation(K)[:n_inf]] = math.inf
    th = rng.normal(size=(K, D)) * 3 + 1
    floor = np.full(D, 1e-3)
    rc, mu, var, e, dg = orc.cem_update(J, th, Ke, floor, 1, np.ones(D))
    fin = np.flatnonzero(np.isfinite(J))
    assert rc == 0 and dg.n_diverged == n_inf
    np.testing.assert_array_equal(e, np.argsort(J, kind="stable")[:Ke])
    sel = fin[np.argsort(J[fin], kind="stable")][:Ke]
    np.testing.assert_allclose(mu, th[sel].mean(0), rtol=0, atol=1e-12)
    np.testing.assert_allclose(var, np.maximum(th[sel].var(0), floor), rtol=0, atol=1e-12)
    assert dg.omega == len(sel)
