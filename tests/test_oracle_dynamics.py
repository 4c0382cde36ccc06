"""Pins for the SRBD model Eq. 1 (O10) and its RK4 discretisation
(O11, reading L25): SPEC's worked cases, the textbook forward Euler-rate
map, scipy's rotation for R, an independent high-order ODE solver, and rigid
body invariants."""
import json
import math
import os

import numpy as np
import pytest
from scipy.integrate import solve_ivp
from scipy.spatial.transform import Rotation

from paper_2403_11383_b200.workloads import HIPS, base_config

GOLD = os.path.join(os.path.dirname(__file__), "golden")
PV = json.load(open(os.path.join(GOLD, "paper_values.json")))


def _cfg(**kw):
    c = base_config()
    c.update(mass=21.0, inertia=[0.135, 0, 0, 0, 0.54, 0, 0, 0, 0.58], gravity=[0, 0, -9.81])
    c.update(kw)
    return c


def test_free_fall(orc):
    ff = PV["free_fall"]
    cfg = _cfg()
    x = np.zeros(12)
    x[2] = 0.35
    xd = orc.dynamics(cfg, x, np.zeros(12), [0, 0, 0, 0], np.zeros(12))
    np.testing.assert_allclose(xd, [0, 0, 0, 0, 0, -9.81, 0, 0, 0, 0, 0, 0], atol=1e-15)
    xn = orc.rk4(cfg, x, np.full(12, 77.0), [0, 0, 0, 0], np.zeros(12), ff["dt"])  # swing: forces ignored
    assert xn[5] == pytest.approx(ff["v_z"], abs=1e-15)
    assert xn[2] - 0.35 == pytest.approx(ff["dz"], abs=1e-15)


def test_static_hover(orc):
    cfg = _cfg()
    x = np.zeros(12)
    x[2] = 0.35
    feet = np.concatenate([HIPS[i] for i in range(4)])
    fz = PV["hover_force"]["fz"]
    assert 21.0 * 9.81 / 4 == pytest.approx(fz)
    gam = np.tile([0, 0, fz], 4)
    xd = orc.dynamics(cfg, x, gam, [1, 1, 1, 1], feet)
    np.testing.assert_allclose(xd, 0.0, atol=1e-12)
    xs = x.copy()
    for _ in range(100):
        xs = orc.rk4(cfg, xs, gam, [1, 1, 1, 1], feet, 0.02)
    np.testing.assert_allclose(xs, x, atol=1e-9)


def test_single_foot_torque(orc):
    sf = PV["single_foot_torque"]
    cfg = _cfg(inertia=[sf["inertia_diag"][0], 0, 0, 0, sf["inertia_diag"][1], 0, 0, 0, sf["inertia_diag"][2]])
    x = np.zeros(12)
    feet = np.zeros(12)
    feet[0:3] = sf["p_cf"]           # p_c = 0 so p_f = p_cf
    gam = np.zeros(12)
    gam[0:3] = sf["Gamma"]
    xd = orc.dynamics(cfg, x, gam, [1, 0, 0, 0], feet)
    np.testing.assert_allclose(xd[9:12], sf["wdot"], atol=1e-12)


def _E_forward(phi, th):
    # body rates from ZYX Euler rates (textbook): w = E'(Phi) Phi_dot
    return np.array([[1, 0, -math.sin(th)],
                     [0, math.cos(phi), math.sin(phi) * math.cos(th)],
                     [0, -math.sin(phi), math.cos(phi) * math.cos(th)]])


def test_euler_rate_map_inverse(orc):
    cfg = _cfg()
    rng = np.random.default_rng(8)
    for _ in range(100):
        x = np.zeros(12)
        x[6:9] = [rng.uniform(-1, 1), rng.uniform(-1, 1), rng.uniform(-3, 3)]
        x[9:12] = rng.normal(size=3)
        xd = orc.dynamics(cfg, x, np.zeros(12), [0] * 4, np.zeros(12))
        np.testing.assert_allclose(_E_forward(x[6], x[7]) @ xd[6:9], x[9:12], atol=1e-12)
    x = np.zeros(12)
    x[9:12] = [0.3, -0.2, 0.7]
    np.testing.assert_allclose(orc.dynamics(cfg, x, np.zeros(12), [0] * 4, np.zeros(12))[6:9], x[9:12], atol=1e-15)


def test_rotation_against_scipy(orc):
    # with w = 0: I w_dot = R^T tau_world; R from scipy's intrinsic ZYX Euler angles
    rng = np.random.default_rng(9)
    I = np.array([[0.2, 0.01, -0.02], [0.01, 0.5, 0.03], [-0.02, 0.03, 0.6]])
    cfg = _cfg(inertia=list(I.ravel()))
    for _ in range(50):
        x = np.zeros(12)
        x[0:3] = rng.normal(size=3) * 0.1
        ang = [rng.uniform(-1, 1), rng.uniform(-1, 1), rng.uniform(-3, 3)]
        x[6:9] = ang
        feet = rng.normal(size=12) * 0.3
        gam = rng.normal(size=12) * 40
        st = [1, 0, 1, 1]
        xd = orc.dynamics(cfg, x, gam, st, feet)
        R = Rotation.from_euler("ZYX", [ang[2], ang[1], ang[0]]).as_matrix()
        tau = sum(np.cross(feet[3 * i:3 * i + 3] - x[0:3], gam[3 * i:3 * i + 3]) for i in range(4) if st[i])
        np.testing.assert_allclose(I @ xd[9:12], R.T @ tau, atol=1e-10)
        F = sum(gam[3 * i:3 * i + 3] for i in range(4) if st[i])
        np.testing.assert_allclose(xd[3:6], F / 21.0 + np.array([0, 0, -9.81]), atol=1e-12)
        np.testing.assert_allclose(xd[0:3], x[3:6], atol=0)


def test_linearity_in_forces(orc):
    cfg = _cfg()
    rng = np.random.default_rng(10)
    x = rng.normal(size=12) * 0.2
    feet = rng.normal(size=12) * 0.3
    g1, g2 = rng.normal(size=12) * 30, rng.normal(size=12) * 30
    st = [1, 1, 0, 1]
    d = lambda g: orc.dynamics(cfg, x, g, st, feet)
    np.testing.assert_allclose(d(g1 + g2), d(g1) + d(g2) - d(np.zeros(12)), atol=1e-10)


def test_rk4_against_independent_solver(orc):
    cfg = _cfg()
    rng = np.random.default_rng(11)
    for _ in range(20):
        x = np.zeros(12)
        x[0:3] = [0.01, -0.02, 0.35]
        x[3:6] = rng.normal(size=3) * 0.3
        x[6:9] = rng.normal(size=3) * 0.1
        x[9:12] = rng.normal(size=3) * 0.5
        feet = np.concatenate([HIPS[i] for i in range(4)]) + rng.normal(size=12) * 0.02
        gam = np.tile([0, 0, 51.5], 4) + rng.normal(size=12) * 3
        st = [1, 0, 0, 1]
        rhs = lambda t, y: orc.dynamics(cfg, y, gam, st, feet)
        ref = solve_ivp(rhs, (0, 0.02), x, method="DOP853", rtol=1e-13, atol=1e-13).y[:, -1]
        got = orc.rk4(cfg, x, gam, st, feet, 0.02)
        assert np.max(np.abs(got - ref)) < 1e-5                 # S:84 (our torques are larger)
        # the local error of RK4 is O(h^5): halving h cuts it ~32x
        half = orc.rk4(cfg, orc.rk4(cfg, x, gam, st, feet, 0.01), gam, st, feet, 0.01)
        assert np.max(np.abs(half - ref)) < np.max(np.abs(got - ref)) / 8 + 1e-13


def test_torque_free_energy_and_momentum(orc):
    I = np.diag([0.135, 0.54, 0.58])
    cfg = _cfg()
    x = np.zeros(12)
    x[9:12] = [0.4, 0.3, -0.5]
    x[6:9] = [0.1, -0.2, 0.3]
    E0 = 0.5 * x[9:12] @ I @ x[9:12]
    def Lw(xx):
        R = Rotation.from_euler("ZYX", [xx[8], xx[7], xx[6]]).as_matrix()
        return R @ (I @ xx[9:12])
    L0 = Lw(x)
    for _ in range(1000):
        x = orc.rk4(cfg, x, np.zeros(12), [0] * 4, np.zeros(12), 0.02)
        assert abs(x[7]) < 1.4
    assert abs(0.5 * x[9:12] @ I @ x[9:12] - E0) / E0 < 1e-6
    np.testing.assert_allclose(Lw(x), L0, atol=1e-5)              # world-frame angular momentum
