"""Pins for the GRF spline (O8, reading L7) and the friction cone
(O9, reading L9): polynomial reproduction, interpolation, the
Catmull-Rom midpoint rule, C1 continuity, and SPEC's worked cone cases."""
import json
import os

import numpy as np
import pytest

from paper_2403_11383_b200.workloads import base_config

GOLD = os.path.join(os.path.dirname(__file__), "golden")


@pytest.mark.parametrize("P", [2, 3, 4, 5, 8])
def test_constant_and_linear_reproduction(orc, P):
    for den in (7, 10, 12):
        for num in range(0, (P - 1) * den + 1):
            assert abs(orc.spline_eval([3.5] * P, num, den) - 3.5) < 1e-12
            kn = [2.0 - 0.75 * p for p in range(P)]            # linear data, all segments (L7 phantoms)
            tau = num / den
            assert abs(orc.spline_eval(kn, num, den) - (2.0 - 0.75 * tau)) < 1e-12


@pytest.mark.parametrize("P", [4, 5, 8])
def test_quadratic_reproduction_interior(orc, P):
    q = lambda t: 0.3 * t * t - 1.1 * t + 2.0
    kn = [q(p) for p in range(P)]
    den = 9
    for num in range(den, (P - 2) * den + 1):                   # interior segments s = 1..P-3
        assert abs(orc.spline_eval(kn, num, den) - q(num / den)) < 1e-12


def test_interpolates_knots_and_midpoint_rule(orc):
    rng = np.random.default_rng(5)
    kn = list(rng.normal(size=6))
    for p in range(6):
        assert orc.spline_eval(kn, p * 11, 11) == pytest.approx(kn[p], abs=1e-14)
    # Catmull-Rom at the middle of segment s: (-k[s-1] + 9 k[s] + 9 k[s+1] - k[s+2]) / 16
    for s in range(1, 4):
        want = (-kn[s - 1] + 9 * kn[s] + 9 * kn[s + 1] - kn[s + 2]) / 16
        assert orc.spline_eval(kn, 2 * s + 1, 2) == pytest.approx(want, abs=1e-13)


def test_c1_continuity(orc):
    rng = np.random.default_rng(6)
    kn = list(rng.normal(size=5))
    den = 10 ** 6
    for p in range(1, 4):
        left = (orc.spline_eval(kn, p * den, den) - orc.spline_eval(kn, p * den - 1, den)) * den
        right = (orc.spline_eval(kn, p * den + 1, den) - orc.spline_eval(kn, p * den, den)) * den
        assert abs(left - right) < 1e-4
        # Catmull-Rom tangent at an interior knot = central difference
        assert abs(left - (kn[p + 1] - kn[p - 1]) / 2) < 1e-4


def test_spline_step_layout(orc):
    cfg = base_config(knots=4, horizon=12)
    theta = np.arange(48, dtype=np.float64)
    # at j = 0 every channel equals knot 0: d = leg*3 + axis
    g0 = orc.spline_step(cfg, theta, 0)
    np.testing.assert_array_equal(g0, theta[:12])
    # j = 4 -> tau = 4*3/12 = 1 -> knot 1
    np.testing.assert_allclose(orc.spline_step(cfg, theta, 4), theta[12:24], atol=1e-12)


def test_cone_worked_cases(orc):
    g = json.load(open(os.path.join(GOLD, "paper_values.json")))["cone"]
    cfg = base_config()
    for raw, want in g["cases"]:
        out, pen = orc.cone(cfg, raw)
        np.testing.assert_allclose(out, want, atol=1e-12)
    assert orc.cone(cfg, [10, -10, 100])[1] == 0.0
    assert orc.cone(cfg, [120, 0, 100])[1] == pytest.approx(70.0 ** 2)          # |fx| - mu fz
    assert orc.cone(cfg, [0, 0, -30])[1] == pytest.approx(35.0 ** 2)            # fz_min - fz
    assert orc.cone(cfg, [0, 0, 200])[1] == pytest.approx(20.0 ** 2)            # fz - fz_max
    _, pen = orc.cone(cfg, [0, 0, 1])     # fz 1 -> 5; l = 2.5; |f_x|=0 ok
    assert pen == pytest.approx(16.0)


def test_cone_membership_and_idempotence(orc):
    cfg = base_config()
    rng = np.random.default_rng(7)
    for _ in range(500):
        raw = rng.normal(0, 80, 3)
        out, pen = orc.cone(cfg, raw)
        assert cfg["fz_min"] <= out[2] <= cfg["fz_max"]
        assert abs(out[0]) <= cfg["mu"] * out[2] + 1e-12 and abs(out[1]) <= cfg["mu"] * out[2] + 1e-12
        out2, pen2 = orc.cone(cfg, out)
        assert np.array_equal(out, out2) and pen2 == 0.0
        assert (pen == 0.0) == np.array_equal(out, raw)
