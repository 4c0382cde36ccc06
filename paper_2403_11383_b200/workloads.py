"""Seeded synthetic workloads (configs and per-robot inputs) for tests and bench.

This module is the ONLY code shared by the oracle side (tests, cpu baseline)
and the CUDA side.  It holds none of the method's arithmetic: it only picks
configuration numbers and draws scenario inputs (initial state, gait phase,
feet, reference trajectory) from seeded numpy generators.  The recipe is
DESIGN.md section 6.

Every real number is rounded to binary32 here, so that the oracle (binary64)
and the CUDA path (binary32) receive numerically identical inputs.
"""
from __future__ import annotations

import copy

import numpy as np

SEED = 0x0000000240311383
HIPS = np.array([[0.24, 0.11, 0.0], [0.24, -0.11, 0.0],     # FL, FR
                 [-0.24, 0.11, 0.0], [-0.24, -0.11, 0.0]])  # RL, RR  (L29)
H_NOM = 0.35  # nominal CoM height (L13)


def f32(x):
    """Round a scalar or array to binary32 and return python float(s) / float64 array."""
    a = np.asarray(x, dtype=np.float32).astype(np.float64)
    return float(a) if a.ndim == 0 else a


def base_config(**kw) -> dict:
    """Defaults shared by all configs (readings L9, L11, L19, L22, L29)."""
    Q = np.array([1500, 1500, 3000, 200, 200, 200, 500, 500, 500, 20, 20, 20], dtype=np.float64) * 1e-2
    cfg = dict(
        mass=21.0, inertia=[0.135, 0, 0, 0, 0.54, 0, 0, 0, 0.58], gravity=[0.0, 0.0, -9.81],
        mu=0.5, fz_min=5.0, fz_max=180.0,
        horizon=12, dt=0.02, knots=4,
        duty_factor=0.65, phase_offset=[0.0, 0.5, 0.5, 0.0],
        freq_hz=[1.3, 2.0, 2.4], gait_adapt=0,
        Q=list(Q), R=[1e-6] * 12, rho=0.1, f_nominal=1.3, w_fc=1e-3,
        mode="mppi", n_samples=10000, n_elite=1, **{"lambda": 1.0},
        sigma=[8.0, 8.0, 15.0], sigma_min_frac=0.1,
        elite_preserve=1, warm_shift=1, seed=SEED,
        n_robots=1, sigma_scale=[1.0],
    )
    cfg.update(kw)
    return round_config(cfg)


def round_config(cfg: dict) -> dict:
    out = copy.deepcopy(cfg)
    for k, v in cfg.items():
        if k in ("horizon", "knots", "gait_adapt", "mode", "n_samples", "n_elite", "elite_preserve",
                 "warm_shift", "seed", "n_robots"):
            continue
        if isinstance(v, (list, tuple, np.ndarray)):
            out[k] = [float(t) for t in f32(np.asarray(v, dtype=np.float64))]
        else:
            out[k] = f32(v)
    return out


def initial_distribution(cfg: dict):
    """Gravity-compensating mean (0, 0, mg/4) per leg and knot; var = sigma^2 (L19)."""
    D = 12 * cfg["knots"]
    mean = np.zeros(D)
    fz = f32(cfg["mass"] * -cfg["gravity"][2] / 4.0)
    for d in range(D):
        mean[d] = fz if d % 3 == 2 else 0.0
    var = f32(np.array([cfg["sigma"][d % 3] ** 2 for d in range(D)]))
    st = dict(mean=f32(mean), var=var, freq_idx=0, iter=0)
    if cfg.get("full_cov", 0):                   # C = diag(sigma^2): L = diag(sigma)
        st["chol"] = np.diag(np.sqrt(var))
    return st


def robot_input(cfg: dict, robot: int, cmd=(0.0, 0.0, 0.0), phase=0, push=None, perturb=True,
                seed=SEED) -> dict:
    """Scenario input for one robot: x0, Q0.32 phase, feet_cur/next, x^r (L13, L23)."""
    H, dt = cfg["horizon"], cfg["dt"]
    rng = np.random.default_rng([seed & 0xFFFFFFFF, seed >> 32, robot])
    cmd = np.asarray(cmd, dtype=np.float64)
    x0 = np.zeros(12)
    x0[2] = H_NOM
    x0[3:6] = cmd
    if perturb:
        sd = np.array([5e-3] * 3 + [5e-2] * 3 + [0.02] * 3 + [0.1] * 3)
        x0 += rng.normal(0.0, 1.0, 12) * sd
    if push is not None:                      # emulated push (config 3): v_y, roll
        x0[4] += push[0]
        x0[6] += push[1]
    x0 = f32(x0)
    feet_cur = np.zeros(12)
    for i in range(4):
        feet_cur[3 * i:3 * i + 3] = HIPS[i] + np.array([x0[0], x0[1], 0.0])
    t_st = cfg["duty_factor"] / cfg["f_nominal"]
    feet_next = feet_cur.copy()
    for i in range(4):
        feet_next[3 * i:3 * i + 2] += 0.5 * t_st * cmd[:2]
    xref = np.zeros((H, 12))
    for j in range(H):
        xref[j, 0:2] = x0[0:2] + cmd[:2] * j * dt
        xref[j, 2] = H_NOM
        xref[j, 3:6] = cmd
        xref[j, 8] = x0[8]
    return dict(x0=x0, phase=int(phase) & 0xFFFFFFFF, feet_cur=f32(feet_cur), feet_next=f32(feet_next),
                xref=f32(xref))


def loop_config() -> dict:
    """Closed-loop constants (L38, L40): hip offsets (L29), nominal
    height (L13), fall criterion |roll|, |pitch| > 0.8 rad or p_z < 0.12 m."""
    return dict(hip=f32(HIPS.reshape(12)), h_nom=f32(H_NOM), fall_angle=f32(0.8), fall_height=f32(0.12))


def q32(frac: float) -> int:
    return int(round(frac * 2 ** 32)) & 0xFFFFFFFF


# ---------------------------------------------------------------------------
# BASELINE.json configs
# ---------------------------------------------------------------------------
def config1():
    """single MPPI iteration, trot, N=64 samples, horizon 10."""
    cfg = base_config(n_samples=64, horizon=10, mode="mppi")
    return cfg, [robot_input(cfg, 0)]


def config2(K=10000):
    """MPPI at paper settings: K = 10k, H = 12, dt = 0.02, fixed trot."""
    cfg = base_config(n_samples=K, mode="mppi")
    return cfg, [robot_input(cfg, 0, cmd=(0.5, 0.0, 0.0), phase=q32(0.3))]


def config3(mode="cem", K=10000):
    """CEM (K_e = 1000) or Naive (K_e = 1) with gait-frequency adaptation; pushed x0."""
    ke = 1000 if mode == "cem" else 1
    cfg = base_config(n_samples=K, n_elite=ke, mode=mode, gait_adapt=1)
    return cfg, [robot_input(cfg, 0, cmd=(0.0, 0.1, 0.0), push=(0.5, 0.08))]


def config4(K):
    """large-batch MPPI sweep, same scenario as config 2."""
    return config2(K)


def config5(R=4096, M=1024, seed=SEED):
    """R independent robots x M samples each (batched MPPI)."""
    cfg = base_config(n_samples=M, mode="mppi", n_robots=R)
    rng = np.random.default_rng([seed & 0xFFFFFFFF, 5])
    phases = rng.integers(0, 2 ** 32, size=R, dtype=np.uint64)
    cmds = rng.uniform(-0.5, 0.5, size=(R, 2))
    inputs = [robot_input(cfg, r, cmd=(cmds[r, 0], cmds[r, 1], 0.0), phase=int(phases[r])) for r in range(R)]
    return cfg, inputs
