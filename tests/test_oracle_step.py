"""Pins for one whole iteration (Alg. 5): zero-noise rollout equals
the deterministic SRBD integration (north star), warm-start of constant knots
(S:389), elite preservation, u0 from the new mean, error paths, determinism."""
import math

import numpy as np
import pytest

from paper_2403_11383_b200 import workloads as W


def _state(cfg):
    return W.initial_distribution(cfg)


def test_zero_noise_rollout_equals_deterministic_integration(orc):
    cfg, inputs = W.config1()
    st = _state(cfg)
    st["var"] = np.zeros_like(st["var"])
    inp = inputs[0]
    mu_shift = orc.warm_shift(cfg, st["mean"])
    r = orc.step(cfg, 0, inp, st)
    J_det = orc.rollout(cfg, inp["x0"], inp["phase"], inp["feet_cur"], inp["feet_next"], inp["xref"], mu_shift, 0)
    np.testing.assert_array_equal(r.J, np.full(cfg["n_samples"], J_det))
    np.testing.assert_allclose(r.mean, mu_shift, atol=1e-12)


def test_warm_shift_constant_and_linear(orc):
    cfg = W.base_config()
    mu = W.initial_distribution(cfg)["mean"]
    np.testing.assert_allclose(orc.warm_shift(cfg, mu), mu, atol=1e-12)
    # knots linear in time: shift by dt adds slope*dt, except the clamped last knot
    P, H, dt = cfg["knots"], cfg["horizon"], cfg["dt"]
    T = H * dt
    lin = np.zeros(12 * P)
    for p in range(P):
        lin[p * 12:(p + 1) * 12] = 10.0 + 50.0 * (p * T / (P - 1))
    sh = orc.warm_shift(cfg, lin)
    for p in range(P - 1):
        np.testing.assert_allclose(sh[p * 12:(p + 1) * 12], 10.0 + 50.0 * (p * T / (P - 1) + dt), atol=1e-9)
    np.testing.assert_allclose(sh[(P - 1) * 12:], lin[(P - 1) * 12:], atol=1e-12)


def test_step_outputs_and_determinism(orc):
    cfg, inputs = W.config1()
    s1, s2 = _state(cfg), _state(cfg)
    r1 = orc.step(cfg, 0, inputs[0], s1)
    r2 = orc.step(cfg, 0, inputs[0], s2)
    assert r1.status == 0
    for a in ("mean", "J", "z", "theta", "u0"):
        np.testing.assert_array_equal(getattr(r1, a), getattr(r2, a))
    assert s1["iter"] == 1
    # elite preservation: sample 0 is the shifted mean with zero noise
    assert np.all(r1.z[0] == 0)
    # u0 = delta_0-masked cone projection of knot 0 of the new mean
    for i in range(4):
        if r1.contact0[i]:
            want, _ = orc.cone(cfg, r1.mean[3 * i:3 * i + 3])
            np.testing.assert_allclose(r1.u0[3 * i:3 * i + 3], want, atol=0)
        else:
            assert np.all(r1.u0[3 * i:3 * i + 3] == 0)
    # MPPI weights: the new mean is a convex combination of the samples
    assert np.all(r1.mean <= r1.theta.max(0) + 1e-9) and np.all(r1.mean >= r1.theta.min(0) - 1e-9)
    # next iteration draws fresh noise
    r3 = orc.step(cfg, 0, inputs[0], s1)
    assert not np.array_equal(r3.z[1:], r1.z[1:])


def test_naive_and_cem_steps(orc):
    cfg, inputs = W.config3("naive", K=256)
    st = _state(cfg)
    r = orc.step(cfg, 0, inputs[0], st)
    b = int(np.argmin(r.J))
    np.testing.assert_array_equal(r.mean, r.theta[b])            # theta*
    assert r.freq_idx == r.fidx[b]
    np.testing.assert_array_equal(r.var, _state(cfg)["var"])      # C unchanged
    cfg, inputs = W.config3("cem", K=512)
    cfg["n_elite"] = 50
    st = _state(cfg)
    r = orc.step(cfg, 0, inputs[0], st)
    sel = np.argsort(r.J, kind="stable")[:50]
    np.testing.assert_array_equal(r.elite, sel)
    np.testing.assert_allclose(r.mean, r.theta[sel].mean(0), atol=1e-12)
    floor = (cfg["sigma_min_frac"] * np.array([cfg["sigma"][d % 3] for d in range(48)])) ** 2
    np.testing.assert_allclose(r.var, np.maximum(r.theta[sel].var(0), floor), atol=1e-9)
    assert set(np.unique(r.fidx)) <= {0, 1, 2}


def test_error_paths(orc):
    cfg, inputs = W.config1()
    inp = dict(inputs[0])
    x0 = inp["x0"].copy()
    x0[7] = math.pi / 2 - 1e-4
    st = _state(cfg)
    assert orc.step(cfg, 0, dict(inp, x0=x0), st).status == -2
    x0[7] = math.nan
    assert orc.step(cfg, 0, dict(inp, x0=x0), st).status == -3
    assert st["iter"] == 0
    x0 = inp["x0"].copy()
    x0[3] = 1e8                                                    # every rollout diverges
    r = orc.step(cfg, 0, dict(inp, x0=x0), st)
    assert r.status == 1 and r.n_diverged == cfg["n_samples"]
    np.testing.assert_array_equal(r.mean, _state(cfg)["mean"])     # kept (L27)


def test_config1_regression_fixture(orc):
    import json
    import os
    g = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "config1_oracle.json")))
    cfg, inputs = W.config1()
    st = _state(cfg)
    for s in g["steps"]:
        r = orc.step(cfg, 0, inputs[0], st)
        assert r.status == s["status"] and r.freq_idx == s["freq_idx"]
        np.testing.assert_array_equal(r.J, s["J"])
        np.testing.assert_array_equal(r.mean, s["mean"])
        np.testing.assert_array_equal(r.z[1].view("uint32"), s["z_bits_row1"])
