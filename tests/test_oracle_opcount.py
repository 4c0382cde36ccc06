"""Pins for the oracle's op-counting mode (oracle/opcount.cpp; the
roofline's algorithmic FLOPs are frozen "by running the oracle in op-counting mode
over the config-2 workload").

The counting build runs the unchanged oracle source with counting scalars, so
(i) its results must equal the plain oracle's bit for bit, and (ii) its counts
must equal closed forms written out by hand from the structure of the method:
  * one evaluation of Eq. 1 with n stance legs, diagonal inertia and
    g = (0, 0, g_z): R = Rz Ry Rx from the sines and cosines (18 FLOPs: the zero
    and one entries of the elementary rotations are identities), per stance leg
    lever arm (3), r x Gamma (9) and the force / torque sums (6; the first leg's
    6 are identities), I w (3), w x I w (9), R^T tau (15), tau - w x I w (3),
    I^-1 (.) (3), F / m + g (4), E'^-1 w (5 + 3 + 4): 61 + 18 n;
  * RK4: 4 evaluations + 3 stage states (2 x 12 each) + the combination
    (7 x 12) = 4 (61 + 18 n) + 156;
  * the Catmull-Rom spline, per channel and step: 7 when the
    evaluation point is inside a segment, 0 on a knot, + 2 for each phantom end
    knot the segment needs (computed even when its weight is zero);
  * cone (L9) 11 per stance leg, penalty sum n - 1, tracking cost 12 x 3 + 11,
    effort (L12) 10 per stance leg, w_fc pen 2, J += stage (not at j = 0);
so one horizon step costs 448 + 94 n_j + 12 spline_j + [j > 0], and the rollout
adds 1 for rho (f - f_n)^2 when f != f_n.
"""
import math

import numpy as np
import pytest

from paper_2403_11383_b200 import workloads as W
from test_oracle_rollout import _cfg, _hover_inputs

M, G = 21.0, 9.81


def _spline_flops(P, H, j):
    a = j * (P - 1)
    s, u_num = a // H, a % H
    if s >= P - 1:
        s, u_num = P - 2, 1
    return 7 * (u_num != 0) + 2 * (s == 0) + 2 * (s == P - 2)


def _rollout_closed_form(orc, cfg, phase0, fidx):
    H, P = cfg["horizon"], cfg["knots"]
    d = orc.contact_sequence(cfg, phase0, cfg["freq_hz"][fidx]).reshape(H, 4)
    n = d.sum(1)
    assert n.min() >= 1
    tot = sum(448 + 94 * int(n[j]) + 12 * _spline_flops(P, H, j) + (j > 0) for j in range(H))
    return tot + (cfg["freq_hz"][fidx] != cfg["f_nominal"])


@pytest.mark.parametrize("duty,off,H,P,fidx,phase", [
    (1.0, [0, 0, 0, 0], 12, 4, 0, 0),
    (0.5, [0, .5, .5, 0], 12, 4, 0, 0),
    (0.65, [0, .5, .5, 0], 12, 4, 0, W.q32(0.3)),      # the config-2 schedule
    (0.65, [0, .5, .5, 0], 10, 4, 2, W.q32(0.7)),
    (0.65, [0, 0, .5, .5], 16, 6, 1, 12345),            # pace-like offsets, P = 6
    (0.8, [0, .25, .5, .75], 12, 3, 2, 99),
])
def test_rollout_count_closed_form(orc, duty, off, H, P, fidx, phase):
    cfg = _cfg(duty_factor=duty, phase_offset=off, horizon=H, knots=P)
    x0, feet, xref = _hover_inputs(H)
    rng = np.random.default_rng(H * P + fidx)
    x0 = x0 + rng.normal(size=12) * 0.01
    feet = feet + rng.normal(size=12) * 0.01
    xref = xref + rng.normal(size=xref.shape) * 0.01
    for trial in range(3):
        th = np.tile([0, 0, M * G / 4], 4 * P) + rng.normal(size=12 * P) * np.tile([8, 8, 15], 4 * P)
        J = orc.rollout(cfg, x0, phase, feet, feet, xref, th, fidx)
        Jc, fl, tr, _ = orc.count_rollout(cfg, x0, phase, feet, feet, xref, th, fidx)
        assert math.isfinite(J)
        assert Jc == J                                   # same arithmetic, same bits
        assert fl == _rollout_closed_form(orc, cfg, phase, fidx)
        assert tr == H * (4 * 7 + 1)                     # 3 sincos + tan per evaluation, yaw wrap


def test_sample_count_closed_form(orc):
    """Normative binary32 Box-Muller per pair: ln 18 (+1 when the
    mantissa is halved, m > sqrt 2), radius 1, sincos 22, z 2; theta2 = mu' + sigma z:
    2 per coordinate."""
    cfg, _ = W.config2()
    st = W.initial_distribution(cfg)
    mu_shift = orc.warm_shift(cfg, st["mean"])
    D = 12 * cfg["knots"]
    key = [cfg["seed"] & 0xFFFFFFFF, cfg["seed"] >> 32]
    for k in (1, 2, 77, 9999):
        th, fl, tr, _ = orc.count_sample(cfg, mu_shift, st["var"], 0, 5, 0, k)
        th_ref, _, _ = orc.sample(cfg, mu_shift, st["var"], 0, 5, 0, k)
        np.testing.assert_array_equal(th, th_ref)
        n_half = 0
        for q in range(D // 4):
            w = orc.philox([q, k, 5, 0], key)
            for w0 in (int(w[0]), int(w[2])):
                n = 2 * (w0 >> 9) + 1
                m = n / 2.0 ** math.floor(math.log2(n))      # mantissa in [1, 2), exact
                n_half += m > np.float32(math.sqrt(2.0))
        assert fl == (D // 2) * 43 + n_half + 2 * D
        assert tr == D // 2                              # one sqrt per pair


@pytest.mark.parametrize("lam", [1.0, 0.5])
def test_mppi_count_closed_form(orc, lam):
    """O13 as the oracle writes it: J - beta (and / lambda unless lambda = 1), the
    sums Omega, sum w^2 and sum J (first term of each is an identity), the mean of
    the finite costs, w_k / Omega * theta per coordinate, ESS."""
    rng = np.random.default_rng(3)
    K, D = 50, 12
    J = rng.uniform(0, 3, K)
    J[7] = math.inf
    th = rng.normal(size=(K, D))
    mu, fl, tr, _ = orc.count_mppi(J, th, lam)
    _, mu_ref, _ = orc.mppi(J, th, lam)
    np.testing.assert_array_equal(mu, mu_ref)
    n_fin = K - 1
    want = K * (1 + (lam != 1.0)) + (K - 1) + K + (K - 1) + (n_fin - 1) + 1 + D * (3 * K - 1) + 2
    assert fl == want
    assert tr == K


def test_config2_count_is_the_bench_numerator():
    """bench.py's frozen algorithmic FLOPs per sample-step are the op-counting mode's
    config-2 figure (scripts/op_count.py), not a profiler count."""
    import importlib.util
    import os
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, os.path.join(root, "scripts"))
    import op_count
    cfg, inputs = W.config2()
    got = op_count.count(cfg, inputs[0], n=32)["per_sample_step"]
    spec = importlib.util.spec_from_file_location("bench_mod", os.path.join(root, "bench.py"))
    bench = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(bench)
    assert bench.ALG_FLOP_ROLLOUT == pytest.approx(got["rollout_flop"], abs=1e-9)
    assert bench.ALG_FLOP_FUSED == pytest.approx(got["fused_flop"], abs=1.0)
