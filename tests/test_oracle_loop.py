"""Pins of the oracle's closed-loop functions (DESIGN readings L36-L40).

Each check is fixed by something other than the oracle's own formula: a value
printed in the paper / SPEC's hand evaluations, a closed form of the
mechanics, a special case that reduces to an already-pinned routine, the
independent numpy construction of the reference in workloads.py, or the
worked Q0.32 gait table of SURVEY 8(c3).
"""
import json
import math
import os

import numpy as np
import pytest

from paper_2403_11383_b200 import workloads as W

GOLD = os.path.join(os.path.dirname(__file__), "golden")
PV = json.load(open(os.path.join(GOLD, "paper_values.json")))


# ---------------------------------------------------------------------------
# Eq. 3 foothold
# ---------------------------------------------------------------------------
def test_foothold_nominal_hand_value(orc):
    g = PV["foothold_nominal"]
    p = orc.foothold(g["p_hip"], g["v_c"], g["v_d"], g["p_cz"], g["T_st"], g["g"])
    np.testing.assert_allclose(p, g["p_f"], rtol=0, atol=1e-12)


def test_foothold_capture_point_hand_value(orc):
    g = PV["foothold_capture"]
    p = orc.foothold(g["p_hip"], g["v_c"], g["v_d"], g["p_cz"], g["T_st"], g["g"])
    assert abs((p[0] - g["p_hip"][0]) - g["x_offset"]) <= g["tol"]
    assert p[1] == g["p_hip"][1] and p[2] == 0.0


def test_foothold_feedback_direction_and_magnitude(orc):
    """the disturbance term moves along (v_c - v_d) with magnitude sqrt(p_cz/g) |v_c - v_d|."""
    rng = np.random.default_rng(3)
    for _ in range(50):
        hip = np.r_[rng.normal(size=2), 0.0]
        vd = np.r_[rng.normal(size=2), 0.0]
        vc = np.r_[rng.normal(size=2), 0.0]
        pcz, tst = rng.uniform(0.2, 0.5), rng.uniform(0.2, 0.6)
        base = orc.foothold(hip, vd, vd, pcz, tst, 9.81)          # v_c = v_d: feedback term vanishes
        p = orc.foothold(hip, vc, vd, pcz, tst, 9.81)
        d = p - base
        e = vc - vd
        assert abs(np.linalg.norm(d) - math.sqrt(pcz / 9.81) * np.linalg.norm(e)) < 1e-12
        assert np.dot(d, e) >= 0 and abs(d[0] * e[1] - d[1] * e[0]) < 1e-12   # parallel, same sense
        assert p[2] == 0.0


# ---------------------------------------------------------------------------
# plant: Eq. 1 + external wrench, one RK4 control period (L36)
# ---------------------------------------------------------------------------
def _cfg():
    return W.base_config()


def test_plant_zero_wrench_is_the_pinned_rk4(orc):
    cfg = _cfg()
    inp = W.robot_input(cfg, 0, cmd=(0.3, -0.1, 0))
    u = np.array([3.0, -2.0, 60.0, 0, 0, 0, 0, 0, 0, -1.0, 4.0, 45.0])
    st = [1, 0, 0, 1]
    a = orc.plant_step(cfg, inp["x0"], u, st, inp["feet_cur"], np.zeros(6), cfg["dt"])
    b = orc.rk4(cfg, inp["x0"], u, st, inp["feet_cur"], cfg["dt"])
    np.testing.assert_array_equal(a, b)


def test_plant_force_wrench_closed_form(orc):
    """No contact, constant external force: constant acceleration g + F/m, which RK4 integrates exactly."""
    cfg = _cfg()
    x = np.zeros(12)
    x[2] = 0.35
    F = np.array([20.0, -40.0, 10.0])
    h = cfg["dt"]
    xn = orc.plant_step(cfg, x, np.zeros(12), [0] * 4, np.zeros(12), np.r_[F, 0, 0, 0], h)
    a = np.array(cfg["gravity"]) + F / cfg["mass"]
    np.testing.assert_allclose(xn[3:6], a * h, rtol=0, atol=1e-15)
    np.testing.assert_allclose(xn[0:3], x[0:3] + 0.5 * a * h * h, rtol=0, atol=1e-15)
    np.testing.assert_array_equal(xn[6:12], np.zeros(6))


@pytest.mark.parametrize("axis", [0, 1, 2])
def test_plant_torque_about_principal_axis(orc, axis):
    """At rest and level, a world torque along a principal axis gives omega = tau h / I and
    angle = tau h^2 / (2 I) exactly (gyroscopic term and R^T tau stay fixed along that axis)."""
    cfg = _cfg()
    x = np.zeros(12)
    x[2] = 0.35
    tau = np.zeros(3)
    tau[axis] = 7.0
    h = cfg["dt"]
    xn = orc.plant_step(cfg, x, np.zeros(12), [0] * 4, np.zeros(12), np.r_[0, 0, 0, tau], h)
    I = cfg["inertia"][4 * axis]
    assert abs(xn[9 + axis] - tau[axis] * h / I) < 1e-14
    assert abs(xn[6 + axis] - 0.5 * tau[axis] * h * h / I) < 1e-14


def test_plant_torque_is_rotated_into_the_body_frame(orc):
    """Yaw 90 deg: a world-y torque is a body-x torque (catches R vs R^T)."""
    cfg = _cfg()
    x = np.zeros(12)
    x[2] = 0.35
    x[8] = math.pi / 2
    xd = orc.plant_dynamics(cfg, x, np.zeros(12), [0] * 4, np.zeros(12), [0, 0, 0, 0, 5.0, 0])
    Ixx = cfg["inertia"][0]
    np.testing.assert_allclose(xd[9:12], [5.0 / Ixx, 0, 0], rtol=0, atol=1e-12)


# ---------------------------------------------------------------------------
# reference (L13)
# ---------------------------------------------------------------------------
def test_reference_matches_the_workload_construction(orc):
    """workloads.robot_input builds x^r independently in numpy (L13 with yaw rate 0)."""
    cfg = _cfg()
    for cmd in [(0.5, 0, 0), (0, 0.1, 0), (-0.3, 0.2, 0)]:
        inp = W.robot_input(cfg, 2, cmd=cmd)
        xr = orc.reference(cfg, W.H_NOM, inp["x0"], cmd, 0.0)
        np.testing.assert_allclose(xr, inp["xref"], rtol=0, atol=2e-7)    # workloads rounds to binary32


def test_reference_yaw_rate(orc):
    cfg = _cfg()
    x = np.zeros(12)
    x[8] = 0.3
    xr = orc.reference(cfg, 0.35, x, [0, 0, 0], 0.5)
    np.testing.assert_allclose(xr[:, 8], 0.3 + 0.5 * cfg["dt"] * np.arange(cfg["horizon"]), atol=1e-15)
    assert np.all(xr[:, 11] == 0.5)


# ---------------------------------------------------------------------------
# advance: phase, touchdown, fall flag (L37, L38, L40)
# ---------------------------------------------------------------------------
def _advance_n(orc, cfg, lc, inp, n, fidx):
    """n advances with zero plant input change (the contact flags come from the phase)."""
    touch = []
    cur = dict(inp)
    thr = orc.stance_threshold(cfg["duty_factor"])
    offs = [int(round(o * 2 ** 32)) & 0xFFFFFFFF for o in cfg["phase_offset"]]
    for j in range(n):
        contact = [int(((cur["phase"] + offs[i]) & 0xFFFFFFFF) < thr) for i in range(4)]
        u0 = np.zeros(12)
        for i in range(4):
            u0[3 * i + 2] = contact[i] * 60.0
        r = orc.advance(cfg, lc, cur, u0, contact, fidx, (0, 0, 0))
        landed = [not np.array_equal(r.feet_cur[3 * i:3 * i + 3], cur["feet_cur"][3 * i:3 * i + 3]) for i in range(4)]
        touch.append(landed)
        cur = dict(x0=r.x0, phase=r.phase, feet_cur=r.feet_cur, feet_next=r.feet_next + 0.0, xref=r.xref)
        # make every planned foothold distinguishable from the current one
        cur["feet_next"] = cur["feet_next"] + 1.0
    return np.array(touch)


def test_advance_phase_and_touchdown_follow_the_worked_gait_table(orc):
    """SURVEY 8(c3) O7 at phi0 = 0, D_f = 0.65: FR/RL lift off at j = 4 and touch down at
    j = 11 at 2.4 Hz; FL/RR never lift off in the first 12 steps."""
    cfg = _cfg()
    lc = W.loop_config()
    inp = W.robot_input(cfg, 0, perturb=False)
    g = PV["gait_worked_q32"]
    touch = _advance_n(orc, cfg, lc, inp, 12, fidx=2)          # 2.4 Hz
    # advance j (0-based) moves the phase from step j to step j + 1
    landed_at = [j + 1 for j in range(12) if touch[j, 1]]
    assert landed_at == [g["touchdown_step_2p4"]]
    assert [j + 1 for j in range(12) if touch[j, 2]] == [g["touchdown_step_2p4"]]
    assert not touch[:, 0].any() and not touch[:, 3].any()


def test_advance_landing_takes_the_planned_foothold_and_replans_with_eq3(orc):
    cfg = _cfg()
    lc = W.loop_config()
    inp = W.robot_input(cfg, 0, cmd=(0.5, 0, 0), perturb=False)
    inp = dict(inp, phase=W.q32(0.45))                       # FR/RL in swing, about to land
    thr = orc.stance_threshold(cfg["duty_factor"])
    offs = [0, 2 ** 31, 2 ** 31, 0]
    contact = [int(((inp["phase"] + o) & 0xFFFFFFFF) < thr) for o in offs]
    assert contact == [1, 0, 0, 1]
    u0 = np.zeros(12)
    r = None
    cur = inp
    for _ in range(40):                                      # until FR lands
        contact = [int(((cur["phase"] + o) & 0xFFFFFFFF) < thr) for o in offs]
        r = orc.advance(cfg, lc, cur, u0, contact, 0, (0.5, 0, 0))
        if not np.array_equal(r.feet_cur[3:6], cur["feet_cur"][3:6]):
            np.testing.assert_array_equal(r.feet_cur[3:6], cur["feet_next"][3:6])
            break
        cur = dict(x0=r.x0, phase=r.phase, feet_cur=r.feet_cur, feet_next=r.feet_next, xref=r.xref)
    else:
        pytest.fail("FR never landed")
    # the replanned footholds are Eq. 3 at the new state (hip rotated by yaw, projected to z = 0)
    t_st = cfg["duty_factor"] / cfg["freq_hz"][0]
    x = r.x0
    for i in range(4):
        h = lc["hip"][3 * i:3 * i + 3]
        c, s = math.cos(x[8]), math.sin(x[8])
        p_hip = [x[0] + c * h[0] - s * h[1], x[1] + s * h[0] + c * h[1], 0.0]
        np.testing.assert_allclose(r.feet_next[3 * i:3 * i + 3],
                                   orc.foothold(p_hip, [x[3], x[4], 0], [0.5, 0, 0], x[2], t_st, 9.81),
                                   rtol=0, atol=1e-15)


def test_advance_fall_flag(orc):
    cfg = _cfg()
    lc = W.loop_config()
    inp = W.robot_input(cfg, 0, perturb=False)
    contact = [1, 0, 0, 1]
    u0 = np.zeros(12)
    assert orc.advance(cfg, lc, inp, u0, contact, 0, (0, 0, 0)).fallen == 0     # one period of free fall: 2 mm
    low = dict(inp, x0=np.r_[inp["x0"][:2], 0.11, inp["x0"][3:]])
    assert orc.advance(cfg, lc, low, u0, contact, 0, (0, 0, 0)).fallen == 1
    tilt = inp["x0"].copy()
    tilt[6] = 0.81
    assert orc.advance(cfg, lc, dict(inp, x0=tilt), u0, contact, 0, (0, 0, 0)).fallen == 1
    tilt[6], tilt[7] = 0.0, -0.81
    assert orc.advance(cfg, lc, dict(inp, x0=tilt), u0, contact, 0, (0, 0, 0)).fallen == 1


def test_advance_hover_is_a_fixed_point(orc):
    """D_f = 1, feet symmetric about the CoM, u0 = (0, 0, mg/4), at rest: the plant does not move
    (the per-iteration closed form of S:359's perfect hover)."""
    cfg = W.base_config(duty_factor=1.0)
    lc = W.loop_config()
    inp = W.robot_input(cfg, 0, perturb=False)
    fz = cfg["mass"] * 9.81 / 4
    u0 = np.tile([0, 0, fz], 4)
    r = orc.advance(cfg, lc, inp, u0, [1] * 4, 0, (0, 0, 0))
    np.testing.assert_allclose(r.x0, inp["x0"], rtol=0, atol=1e-7)     # inputs carry binary32 rounding
    assert r.fallen == 0
    np.testing.assert_array_equal(r.feet_cur, inp["feet_cur"])       # no touchdown in full stance
