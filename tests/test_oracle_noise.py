"""Pins for the oracle's noise (recipe O1-O6): Philox KAT
vectors, ln / sincos against binary64 libm, Gaussian moments and KS test,
theta1 uniformity.  None of these re-derives the recipe itself."""
import json
import math
import os

import numpy as np
import pytest
from scipy import stats

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def test_philox_kat(orc):
    kat = json.load(open(os.path.join(GOLD, "philox_kat.json")))
    for v in kat["vectors"]:
        ctr = [int(x, 16) for x in v["ctr"]]
        key = [int(x, 16) for x in v["key"]]
        assert orc.philox(ctr, key) == [int(x, 16) for x in v["out"]]


def _edge_words(rng, n):
    w = list(rng.integers(0, 2 ** 32, size=n, dtype=np.uint64))
    w += [0, 1, 0x1FF, 0x200, 0xFFFFFFFF, 0xFFFFFE00, 0x80000000, 0x7FFFFFFF,
          0x20000000, 0x1FFFFFFF, 0x3FFFFE00, 0x5A827999]
    return [int(x) for x in w]


def _ulp32(x):
    x = abs(float(np.float32(x)))
    return float(np.spacing(np.float32(x))) if x > 0 else float(np.float32(1.4e-45))


def test_ln_u24_against_libm(orc):
    rng = np.random.default_rng(1)
    worst = 0.0
    for w in _edge_words(rng, 20000):
        u1 = (2 * (w >> 9) + 1) * 2.0 ** -24
        exact = math.log(u1)
        got = orc.ln_u24(w)
        err = abs(got - exact) / _ulp32(exact)
        worst = max(worst, err)
    assert worst <= 2.5, worst


def test_sincos_2pi_against_libm(orc):
    rng = np.random.default_rng(2)
    worst = 0.0
    words = _edge_words(rng, 20000)
    # both ends of every octant
    for o in range(8):
        words += [(o << 29) | (0 << 9), (o << 29) | (0xFFFFF << 9) | 0x1FF]
    for w in words:
        u2 = ((w >> 9) + 0.5) * 2.0 ** -23
        s, c = orc.sincos_2pi_u(w)
        es, ec = math.sin(2 * math.pi * u2), math.cos(2 * math.pi * u2)
        worst = max(worst, abs(float(s) - es), abs(float(c) - ec))
    assert worst < 1.2e-7, worst          # ~2 ulp of 1.0 in binary32


def test_box_muller_special_words(orc):
    # w0 = 0 -> u1 = 2^-24 -> r = sqrt(48 ln 2); w1 = 0 -> angle ~ 0 -> (z0, z1) ~ (r, 0)
    z = orc.normal4([0, 0, 0xFFFFFFFF, 0x40000000])
    r = math.sqrt(48 * math.log(2))
    assert abs(z[0] - r) < 4e-6 and abs(z[1]) < 1e-5
    # w2 = max -> u1 = 1 - 2^-24 -> r ~ sqrt(2^-23); w3 = 0x40000000 -> angle pi/2 -> (0, r)
    r2 = math.sqrt(-2 * math.log(1 - 2.0 ** -24))
    assert abs(z[3] - r2) < 1e-9 and abs(z[2]) < 1e-9
    assert max(abs(z)) <= 5.77


def test_gaussian_moments_and_ks(orc):
    cfg = __import__("paper_2403_11383_b200.workloads", fromlist=["x"]).base_config(knots=2)
    D = 24
    zs = []
    mu = np.zeros(D)
    var = np.ones(D)
    for k in range(1, 4001):                  # 4000 samples x 24 coordinates = 96k draws
        _, z, _ = orc.sample(cfg, mu, var, 0, 7, 3, k)
        zs.append(z)
    z = np.concatenate(zs).astype(np.float64)
    n = z.size
    assert abs(z.mean()) < 3 / math.sqrt(n)
    # var of the sample variance for a normal is 2/n
    assert abs(z.var() - 1.0) < 3 * math.sqrt(2.0 / n)
    assert stats.kstest(z, "norm").pvalue > 1e-3
    # independence of the pair members: correlation of z0 with z1 small
    zz = np.stack(zs).astype(np.float64)
    assert abs(np.corrcoef(zz[:, 0], zz[:, 1])[0, 1]) < 0.06


def test_theta_scaling_and_elite_preservation(orc):
    from paper_2403_11383_b200.workloads import base_config
    cfg = base_config(knots=4)
    D = 48
    mu = np.linspace(-3, 3, D)
    var = np.linspace(0.5, 4, D)
    th0, z0, i0 = orc.sample(cfg, mu, var, 2, 5, 0, 0)
    assert np.all(z0 == 0) and np.array_equal(th0, mu) and i0 == 2   # sample 0 = mean (L21)
    th, z, i = orc.sample(cfg, mu, var, 2, 5, 0, 17)
    np.testing.assert_allclose(th, mu + np.sqrt(var) * z.astype(np.float64), rtol=0, atol=1e-12)
    assert i == 2                                                         # gait_adapt off
    # same counter -> same noise; different iter / robot / k -> different noise
    _, z_again, _ = orc.sample(cfg, mu, var, 2, 5, 0, 17)
    assert np.array_equal(z, z_again)
    for args in [(6, 0, 17), (5, 1, 17), (5, 0, 18)]:
        _, z2, _ = orc.sample(cfg, mu, var, 2, *args)
        assert not np.array_equal(z, z2)


def test_theta1_uniform_chi2(orc):
    from paper_2403_11383_b200.workloads import base_config
    cfg = base_config(knots=2, gait_adapt=1)
    counts = np.zeros(3)
    for k in range(1, 6001):
        _, _, idx = orc.sample(cfg, np.zeros(24), np.ones(24), 0, 1, 0, k)
        counts[idx] += 1
    chi2 = ((counts - 2000) ** 2 / 2000).sum()
    assert stats.chi2.sf(chi2, 2) > 1e-3, counts


# ---------------------------------------------------------------------------
# multiple Gaussians (DESIGN L41)
# ---------------------------------------------------------------------------
def test_multiple_gaussians_group_structure(orc):
    """Sample k draws with std sigma_scale[k mod G]: the same z as the one-Gaussian draw,
    a zero scale reproduces mu' exactly, a scale s multiplies theta - mu' by s."""
    from paper_2403_11383_b200 import workloads as W
    base = W.base_config(n_samples=64)
    st = W.initial_distribution(base)
    mu_s = orc.warm_shift(base, st["mean"])
    for k in range(1, 40):
        th1, z1, _ = orc.sample(base, mu_s, st["var"], 0, 3, 0, k)
        th, z, _ = orc.sample(dict(base, sigma_scale=[1.0, 0.0, 2.0]), mu_s, st["var"], 0, 3, 0, k)
        np.testing.assert_array_equal(z, z1)
        g = k % 3
        if g == 0:
            np.testing.assert_array_equal(th, th1)
        elif g == 1:
            np.testing.assert_array_equal(th, mu_s)
        else:
            np.testing.assert_allclose(th - mu_s, 2.0 * (th1 - mu_s), rtol=1e-15, atol=1e-12)
    # elite preservation is unaffected
    th0, _, _ = orc.sample(dict(base, sigma_scale=[3.0, 0.5]), mu_s, st["var"], 0, 3, 0, 0)
    np.testing.assert_array_equal(th0, mu_s)


def test_multiple_gaussians_group_variances(orc):
    from paper_2403_11383_b200 import workloads as W
    cfg = W.base_config(n_samples=64, sigma_scale=[0.5, 1.0, 2.0], elite_preserve=0)
    st = W.initial_distribution(cfg)
    mu_s = orc.warm_shift(cfg, st["mean"])
    dev = {0: [], 1: [], 2: []}
    for k in range(3000):
        th, _, _ = orc.sample(cfg, mu_s, st["var"], 0, 0, 0, k)
        dev[k % 3].append((th - mu_s) / np.sqrt(st["var"]))
    for g, s in enumerate([0.5, 1.0, 2.0]):
        v = np.var(np.array(dev[g]))                 # 1000 x 48 standardised deviations
        assert abs(v / s ** 2 - 1.0) < 0.05
