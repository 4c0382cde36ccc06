"""Pins for Rollout (Alg. 2) with the policy of Alg. 5
and the cost of P:342-351 (O12): whole-rollout closed forms (perfect hover,
vertical thrust), single-channel cost, the rho term, sagittal mirror
symmetry, the touchdown foot switch (L23), divergence (L26)."""
import math

import numpy as np
import pytest

from paper_2403_11383_b200.workloads import HIPS, base_config

M, G = 21.0, 9.81


def _cfg(**kw):
    c = base_config()
    c.update(mass=M, inertia=[0.135, 0, 0, 0, 0.54, 0, 0, 0, 0.58], gravity=[0, 0, -G],
             dt=0.02, duty_factor=1.0, f_nominal=1.3, freq_hz=[1.3, 2.0, 2.4],
             Q=[15, 15, 30, 2, 2, 2, 5, 5, 5, 0.2, 0.2, 0.2], R=[1e-6] * 12, rho=0.1, w_fc=1e-3,
             mu=0.5, fz_min=5.0, fz_max=180.0)
    c.update(kw)
    return c


def _hover_inputs(H):
    x0 = np.zeros(12)
    x0[2] = 0.35
    feet = np.concatenate([HIPS[i] for i in range(4)])
    xref = np.tile(x0, (H, 1))
    return x0, feet, xref


def test_perfect_hover_zero_cost(orc):
    cfg = _cfg()
    H, P = cfg["horizon"], cfg["knots"]
    x0, feet, xref = _hover_inputs(H)
    theta = np.tile([0, 0, M * G / 4], 4 * P)
    J = orc.rollout(cfg, x0, 0, feet, feet, xref, theta, 0)
    assert abs(J) < 1e-20


@pytest.mark.parametrize("fz", [20.0, 51.5025, 60.0, 120.0])
def test_vertical_thrust_closed_form(orc, fz):
    cfg = _cfg()
    H, P, dt = cfg["horizon"], cfg["knots"], cfg["dt"]
    x0, feet, xref = _hover_inputs(H)
    theta = np.tile([0, 0, fz], 4 * P)
    J = orc.rollout(cfg, x0, 0, feet, feet, xref, theta, 0)
    a = 4 * fz / M - G
    Qz, Qvz, Rz = cfg["Q"][2], cfg["Q"][5], cfg["R"][2]
    want = sum(Qz * (0.5 * a * (j * dt) ** 2) ** 2 + Qvz * (a * j * dt) ** 2 + 4 * Rz * (fz - M * G / 4) ** 2
               for j in range(H))
    assert J == pytest.approx(want, rel=1e-10, abs=1e-14)


def test_single_channel_cost_and_rho(orc):
    cfg = _cfg(Q=[0] * 6 + [0, 0, 0, 0, 0, 0], R=[0] * 12, w_fc=0.0, rho=2.0)
    Qv = [0.0] * 12
    Qv[7] = 3.0
    cfg["Q"] = Qv
    H, P = cfg["horizon"], cfg["knots"]
    x0, feet, xref = _hover_inputs(H)
    xref = xref.copy()
    xref[:, 7] = 0.1                              # constant pitch error of -0.1 at hover
    theta = np.tile([0, 0, M * G / 4], 4 * P)
    J0 = orc.rollout(cfg, x0, 0, feet, feet, xref, theta, 0)
    assert J0 == pytest.approx(H * 3.0 * 0.01, rel=1e-12)       # S:277 q e^2 per step
    J2 = orc.rollout(cfg, x0, 0, feet, feet, xref, theta, 2)   # 2.4 Hz; D_f = 1 keeps the schedule
    assert J2 - J0 == pytest.approx(2.0 * (2.4 - 1.3) ** 2, rel=1e-12)   # 2.42


def test_yaw_error_is_wrapped(orc):
    cfg = _cfg()
    H, P = cfg["horizon"], cfg["knots"]
    x0, feet, xref = _hover_inputs(H)
    x0 = x0.copy()
    x0[8] = 3.0
    theta = np.tile([1.0, -2.0, M * G / 4], 4 * P)
    xr1 = xref.copy()
    xr1[:, 8] = 3.0 + 0.05
    xr2 = xr1.copy()
    xr2[:, 8] -= 2 * math.pi
    assert orc.rollout(cfg, x0, 0, feet, feet, xr1, theta, 0) == pytest.approx(
        orc.rollout(cfg, x0, 0, feet, feet, xr2, theta, 0), rel=1e-12)


def _mirror_state(x):
    m = x.copy()
    for i in (1, 4, 6, 8, 9, 11):     # y, v_y, roll, yaw, w_x, w_z
        m[..., i] = -m[..., i]
    return m


def _mirror_legs(v):                  # per-leg 3-vectors: swap FL<->FR, RL<->RR, negate y
    v = v.reshape(-1, 4, 3).copy()
    v = v[:, [1, 0, 3, 2], :]
    v[:, :, 1] *= -1
    return v.reshape(-1)


def test_sagittal_mirror_symmetry(orc):
    """Mirroring y and swapping left/right legs (with the trot phase shifted by
    half a cycle) must leave the cost unchanged: catches sign errors in the
    cross products, R^T and E'^-1."""
    rng = np.random.default_rng(12)
    for trial in range(20):
        cfg = _cfg(duty_factor=0.65, phase_offset=[0.0, 0.5, 0.5, 0.0], horizon=16)
        H, P = cfg["horizon"], cfg["knots"]
        x0 = np.zeros(12)
        x0[2] = 0.35
        x0 += rng.normal(size=12) * np.array([0.02] * 3 + [0.2] * 3 + [0.1] * 3 + [0.5] * 3)
        feet = np.concatenate([HIPS[i] for i in range(4)]) + rng.normal(size=12) * 0.02
        feet[2::3] = 0.0
        feet_n = feet + rng.normal(size=12) * 0.05
        feet_n[2::3] = 0.0
        xref = np.tile(x0, (H, 1)) + rng.normal(size=(H, 12)) * 0.05
        theta = np.tile([0, 0, 51.5], 4 * P) + rng.normal(size=12 * P) * np.tile([8, 8, 15], 4 * P)
        ph = int(rng.integers(0, 2 ** 32))
        f = int(trial % 3)
        J = orc.rollout(cfg, x0, ph, feet, feet_n, xref, theta, f)
        Jm = orc.rollout(cfg, _mirror_state(x0), (ph + 2 ** 31) & 0xFFFFFFFF,
                         _mirror_legs(feet), _mirror_legs(feet_n), _mirror_state(xref),
                         _mirror_legs(theta), f)
        assert np.isfinite(J)
        assert Jm == pytest.approx(J, rel=1e-11)


def test_touchdown_switches_feet(orc):
    # 2.4 Hz, phi0 = 0, D_f = 0.65: FR and RL touch down at j = 11; FL never does in H = 20
    cfg = _cfg(duty_factor=0.65, phase_offset=[0.0, 0.5, 0.5, 0.0], horizon=20)
    H, P = cfg["horizon"], cfg["knots"]
    x0, feet, xref = _hover_inputs(H)
    theta = np.tile([2.0, 1.0, 60.0], 4 * P)
    J = orc.rollout(cfg, x0, 0, feet, feet, xref, theta, 2)
    fn = feet.copy()
    fn[0:3] += [0.05, 0.03, 0.0]                  # FL: never touches down -> no effect
    assert orc.rollout(cfg, x0, 0, feet, fn, xref, theta, 2) == J
    fn = feet.copy()
    fn[3:6] += [0.05, 0.03, 0.0]                  # FR: touches down at j = 11 -> used from then on
    J2, tr2 = orc.rollout(cfg, x0, 0, feet, fn, xref, theta, 2, traj=True)
    _, tr = orc.rollout(cfg, x0, 0, feet, feet, xref, theta, 2, traj=True)
    assert J2 != J
    np.testing.assert_array_equal(tr2[:12], tr[:12])              # identical through x_11
    assert np.any(tr2[12] != tr[12])


def test_divergence_is_infinite(orc):
    cfg = _cfg()
    H, P = cfg["horizon"], cfg["knots"]
    x0, feet, xref = _hover_inputs(H)
    theta = np.tile([0, 0, 51.5], 4 * P)
    x = x0.copy()
    x[3] = 1e9
    assert orc.rollout(cfg, x, 0, feet, feet, xref, theta, 0) == math.inf
    x = x0.copy()
    x[10] = 200.0                                # pitch rate drives pitch past pi/2 - 1e-3
    assert orc.rollout(cfg, x, 0, feet, feet, xref, theta, 0) == math.inf


@pytest.mark.parametrize("fz", [20.0, M * G / 2, 120.0, 150.0])
def test_two_leg_trot_thrust_closed_form(orc, fz):
    """u^r = -m g_z / max(1, n_stance) with n_stance = 2 (L12, "(u - u^r)^T R
    (u - u^r)"), and swing legs carry neither force nor effort (P:277 delta_i, P:249
    mask).  Trot (offsets 0, 1/2, 1/2, 0), D_f = 0.5, phi0 = 0, 1.3 Hz, H = 12: the
    FL/RR phase reaches 12 * 0.026 = 0.312 < 0.5 of a cycle, so FL and RR stay in
    stance and FR, RL in swing for the whole horizon.  FL and RR hips are mirror
    images through the CoM, so vertical forces of equal size give zero net torque at
    any height and the body rises or falls straight with a = 2 f_z / m - g (RK4 is
    exact for constant acceleration).  With R_z = 1e-3 the effort term is of the
    same order as the tracking terms, so 'm g / 4 always' or 'count swing legs'
    changes J by > 1e-3 relative."""
    cfg = _cfg(duty_factor=0.5, phase_offset=[0.0, 0.5, 0.5, 0.0], R=[1e-3] * 12)
    H, P, dt = cfg["horizon"], cfg["knots"], cfg["dt"]
    assert H == 12
    d = orc.contact_sequence(cfg, 0, 1.3).reshape(H, 4)
    np.testing.assert_array_equal(d, np.tile([1, 0, 0, 1], (H, 1)))
    x0, feet, xref = _hover_inputs(H)
    theta = np.tile([0, 0, fz], 4 * P)
    J = orc.rollout(cfg, x0, 0, feet, feet, xref, theta, 0)
    a = 2 * fz / M - G
    Qz, Qvz, Rz = cfg["Q"][2], cfg["Q"][5], cfg["R"][2]
    want = sum(Qz * (0.5 * a * (j * dt) ** 2) ** 2 + Qvz * (a * j * dt) ** 2 + 2 * Rz * (fz - M * G / 2) ** 2
               for j in range(H))
    assert J == pytest.approx(want, rel=1e-10, abs=1e-14)
    wrong_mg4 = sum(Qz * (0.5 * a * (j * dt) ** 2) ** 2 + Qvz * (a * j * dt) ** 2 + 2 * Rz * (fz - M * G / 4) ** 2
                    for j in range(H))
    assert abs(wrong_mg4 - want) > 1e-3 * want    # the pin separates the readings


@pytest.mark.parametrize("fz_raw,fz_clamped", [(200.0, 180.0), (260.0, 180.0), (0.0, 5.0), (-40.0, 5.0)])
def test_cone_penalty_enters_cost(orc, fz_raw, fz_clamped):
    """L9 / P:294: the stance force is the cone projection of the raw spline output
    (f_z clamped to [fz_min, fz_max]) and J gains w_fc * (squared violation of the raw
    output) per stance leg and step.  D_f = 1, f_z knots outside the bounds, no
    horizontal force: the motion is the vertical-thrust closed form at the clamped
    force, and the penalty adds w_fc * H * 4 * (f_z - bound)^2."""
    cfg = _cfg(w_fc=1e-3)
    H, P, dt = cfg["horizon"], cfg["knots"], cfg["dt"]
    x0, feet, xref = _hover_inputs(H)
    theta = np.tile([0, 0, fz_raw], 4 * P)
    J = orc.rollout(cfg, x0, 0, feet, feet, xref, theta, 0)
    a = 4 * fz_clamped / M - G
    Qz, Qvz, Rz = cfg["Q"][2], cfg["Q"][5], cfg["R"][2]
    thrust = sum(Qz * (0.5 * a * (j * dt) ** 2) ** 2 + Qvz * (a * j * dt) ** 2
                 + 4 * Rz * (fz_clamped - M * G / 4) ** 2 for j in range(H))
    pen = cfg["w_fc"] * H * 4 * (fz_raw - fz_clamped) ** 2
    assert J == pytest.approx(thrust + pen, rel=1e-10)
    # the penalty weight enters linearly: w_fc = 0 leaves the thrust closed form
    J0 = orc.rollout(_cfg(w_fc=0.0), x0, 0, feet, feet, xref, theta, 0)
    assert J0 == pytest.approx(thrust, rel=1e-10)
