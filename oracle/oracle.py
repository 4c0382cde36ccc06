"""ctypes wrapper of ``liboracle.so`` (oracle/sbs_oracle.c).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Argument marshalling
only: every number is computed in the C oracle.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "sbs_oracle.c")
_HDR = os.path.join(_HERE, "sbs_oracle.h")
_LIB = os.path.join(_HERE, "liboracle.so")
_CNT_SRC = os.path.join(_HERE, "opcount.cpp")
_CNT_LIB = os.path.join(_HERE, "libopcount.so")

MAX_KNOTS = 8
MAX_D = 12 * MAX_KNOTS
MAX_FREQ = 8
MODES = {"mppi": 0, "cem": 1, "naive": 2}


def build_oracle(force: bool = False) -> str:
    """Compile the oracle (gcc, -O2 -ffp-contract=off) if stale."""
    stale = force or not os.path.exists(_LIB) or max(
        os.path.getmtime(_SRC), os.path.getmtime(_HDR)) > os.path.getmtime(_LIB)
    if stale:
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-std=gnu11", "-ffp-contract=off", "-fno-fast-math",
                               "-Wall", "-fPIC", "-shared", "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    stale = force or not os.path.exists(_CNT_LIB) or max(
        os.path.getmtime(_SRC), os.path.getmtime(_HDR), os.path.getmtime(_CNT_SRC)) > os.path.getmtime(_CNT_LIB)
    if stale:  # op-counting mode (opcount.cpp): the same source with counting scalars
        tmp = _CNT_LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["g++", "-O1", "-std=c++17", "-ffp-contract=off", "-fno-fast-math", "-Wall",
                               "-Wno-class-memaccess", "-fPIC", "-shared", "-o", tmp, _CNT_SRC])
        os.replace(tmp, _CNT_LIB)
    return _LIB


class OrcConfig(C.Structure):
    _fields_ = [
        ("mass", C.c_double), ("inertia", C.c_double * 9), ("gravity", C.c_double * 3),
        ("mu", C.c_double), ("fz_min", C.c_double), ("fz_max", C.c_double),
        ("horizon", C.c_int32), ("knots", C.c_int32), ("dt", C.c_double),
        ("duty_factor", C.c_double), ("phase_offset", C.c_double * 4),
        ("n_freq", C.c_int32), ("gait_adapt", C.c_int32), ("freq_hz", C.c_double * MAX_FREQ),
        ("Q", C.c_double * 12), ("R", C.c_double * 12), ("rho", C.c_double),
        ("f_nominal", C.c_double), ("w_fc", C.c_double),
        ("mode", C.c_int32), ("elite_preserve", C.c_int32),
        ("n_samples", C.c_int64), ("n_elite", C.c_int64), ("lambda_", C.c_double),
        ("sigma", C.c_double * 3), ("sigma_min_frac", C.c_double),
        ("warm_shift", C.c_int32), ("_pad", C.c_int32), ("seed", C.c_uint64),
        ("n_sigma_groups", C.c_int32), ("_pad2", C.c_int32), ("sigma_scale", C.c_double * 8),
        ("full_cov", C.c_int32), ("_pad3", C.c_int32),
    ]


class OrcDiag(C.Structure):
    _fields_ = [("j_min", C.c_double), ("j_mean", C.c_double), ("omega", C.c_double),
                ("ess", C.c_double), ("n_diverged", C.c_int64), ("argmin", C.c_int64)]


class OrcState(C.Structure):
    _fields_ = [("mean", C.c_double * MAX_D), ("var", C.c_double * MAX_D),
                ("freq_idx", C.c_int32), ("iter", C.c_uint32), ("chol", C.c_double * (MAX_D * MAX_D))]


class OrcOutput(C.Structure):
    _fields_ = [("u0", C.c_double * 12), ("contact0", C.c_int32 * 4), ("freq_idx", C.c_int32),
                ("status", C.c_int32), ("freq_hz", C.c_double), ("diag", OrcDiag)]


class OrcLoopConfig(C.Structure):
    _fields_ = [("hip", C.c_double * 12), ("h_nom", C.c_double), ("fall_angle", C.c_double),
                ("fall_height", C.c_double)]


def make_loop_config(lc: dict) -> OrcLoopConfig:
    o = OrcLoopConfig()
    o.hip[:] = [float(v) for v in np.asarray(lc["hip"], dtype=np.float64).reshape(12)]
    o.h_nom, o.fall_angle, o.fall_height = float(lc["h_nom"]), float(lc["fall_angle"]), float(lc["fall_height"])
    return o


@dataclass
class AdvanceResult:
    fallen: int
    x0: np.ndarray
    phase: int
    feet_cur: np.ndarray
    feet_next: np.ndarray
    xref: np.ndarray


def _dp(a):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def _f64(a, n=None):
    a = np.ascontiguousarray(np.asarray(a, dtype=np.float64))
    if n is not None:
        assert a.size == n, (a.size, n)
    return a


def make_config(cfg: dict) -> OrcConfig:
    """Build the oracle's own config struct from a workload dict."""
    c = OrcConfig()
    c.mass = cfg["mass"]
    c.inertia[:] = list(np.asarray(cfg["inertia"], dtype=np.float64).ravel())
    c.gravity[:] = list(cfg["gravity"])
    c.mu, c.fz_min, c.fz_max = cfg["mu"], cfg["fz_min"], cfg["fz_max"]
    c.horizon, c.knots, c.dt = cfg["horizon"], cfg["knots"], cfg["dt"]
    c.duty_factor = cfg["duty_factor"]
    c.phase_offset[:] = list(cfg["phase_offset"])
    f = list(cfg["freq_hz"])
    c.n_freq = len(f)
    c.freq_hz[:len(f)] = f
    c.gait_adapt = int(cfg["gait_adapt"])
    c.Q[:] = list(cfg["Q"])
    c.R[:] = list(cfg["R"])
    c.rho, c.f_nominal, c.w_fc = cfg["rho"], cfg["f_nominal"], cfg["w_fc"]
    c.mode = MODES[cfg["mode"]]
    c.elite_preserve = int(cfg["elite_preserve"])
    c.n_samples = cfg["n_samples"]
    c.n_elite = cfg["n_elite"]
    c.lambda_ = cfg["lambda"]
    c.sigma[:] = list(cfg["sigma"])
    c.sigma_min_frac = cfg["sigma_min_frac"]
    c.warm_shift = int(cfg["warm_shift"])
    c.seed = cfg["seed"]
    sc = list(cfg.get("sigma_scale", [1.0]))
    c.n_sigma_groups = len(sc)
    c.sigma_scale[:len(sc)] = [float(v) for v in sc]
    c.full_cov = int(cfg.get("full_cov", 0))
    return c


@dataclass
class StepResult:
    status: int
    mean: np.ndarray
    var: np.ndarray
    freq_idx: int
    freq_hz: float
    u0: np.ndarray
    contact0: np.ndarray
    j_min: float
    j_mean: float
    omega: float
    ess: float
    n_diverged: int
    argmin: int
    J: np.ndarray | None = None
    fidx: np.ndarray | None = None
    theta: np.ndarray | None = None
    z: np.ndarray | None = None
    elite: np.ndarray | None = None


class Oracle:
    """Thin marshalling layer over the C oracle."""

    def __init__(self):
        self.lib = C.CDLL(build_oracle())
        L = self.lib
        u32p, dp, i32p = C.POINTER(C.c_uint32), C.POINTER(C.c_double), C.POINTER(C.c_int32)
        cfgp = C.POINTER(OrcConfig)
        L.orc_philox4x32_10.argtypes = [u32p, u32p, u32p]
        L.orc_ln_u24.argtypes = [C.c_uint32]
        L.orc_ln_u24.restype = C.c_float
        L.orc_sincos_2pi_u.argtypes = [C.c_uint32, C.POINTER(C.c_float), C.POINTER(C.c_float)]
        L.orc_normal4.argtypes = [u32p, C.POINTER(C.c_float)]
        L.orc_normal4_batch.argtypes = [u32p, C.c_int64, C.POINTER(C.c_float)]
        L.orc_sample.argtypes = [cfgp, dp, dp, C.c_int32, C.c_uint32, C.c_uint32, C.c_int64,
                                 dp, C.POINTER(C.c_float), i32p]
        L.orc_warm_shift.argtypes = [cfgp, dp, dp]
        L.orc_phase_inc.argtypes = [C.c_double, C.c_double]
        L.orc_phase_inc.restype = C.c_uint32
        L.orc_stance_threshold.argtypes = [C.c_double]
        L.orc_stance_threshold.restype = C.c_uint64
        L.orc_contact_sequence.argtypes = [cfgp, C.c_uint32, C.c_double, i32p]
        L.orc_spline_eval.argtypes = [C.c_int32, dp, C.c_int64, C.c_int64, dp]
        L.orc_spline_step.argtypes = [cfgp, dp, C.c_int32, dp]
        L.orc_cone.argtypes = [cfgp, dp, dp, dp]
        L.orc_dynamics.argtypes = [cfgp, dp, dp, i32p, dp, dp]
        L.orc_rk4.argtypes = [cfgp, dp, dp, i32p, dp, C.c_double, dp]
        L.orc_rollout.argtypes = [cfgp, dp, C.c_uint32, dp, dp, dp, dp, C.c_int32, dp]
        L.orc_rollout.restype = C.c_double
        L.orc_mppi.argtypes = [C.c_int64, C.c_int32, dp, dp, C.c_double, dp, C.POINTER(OrcDiag)]
        L.orc_cem_select.argtypes = [C.c_int64, dp, C.c_int64, C.POINTER(C.c_int64)]
        L.orc_cem_update.argtypes = [C.c_int64, C.c_int32, dp, dp, C.c_int64, dp, C.c_int32,
                                     dp, dp, C.POINTER(C.c_int64), C.POINTER(OrcDiag)]
        L.orc_step.argtypes = [cfgp, C.c_uint32, dp, C.c_uint32, dp, dp, dp,
                               C.POINTER(OrcState), C.POINTER(OrcOutput), dp, i32p, dp,
                               C.POINTER(C.c_float), C.POINTER(C.c_int64)]
        L.orc_cholesky.argtypes = [C.c_int32, dp, dp]
        L.orc_sample_full.argtypes = [cfgp, dp, dp, C.c_int32, C.c_uint32, C.c_uint32, C.c_int64,
                                      dp, C.POINTER(C.c_float), i32p]
        L.orc_cem_update_full.argtypes = [C.c_int64, C.c_int32, dp, dp, C.c_int64, dp, dp, dp, dp,
                                          C.POINTER(C.c_int64), C.POINTER(OrcDiag)]
        L.orc_foothold.argtypes = [dp, dp, dp, C.c_double, C.c_double, C.c_double, dp]
        L.orc_plant_dynamics.argtypes = [cfgp, dp, dp, i32p, dp, dp, dp]
        L.orc_plant_step.argtypes = [cfgp, dp, dp, i32p, dp, dp, C.c_double, dp]
        L.orc_reference.argtypes = [cfgp, C.c_double, dp, dp, C.c_double, dp]
        L.orc_advance.argtypes = [cfgp, C.POINTER(OrcLoopConfig), dp, C.c_uint32, dp, dp, dp, i32p, C.c_int32,
                                  dp, C.c_double, dp, dp, u32p, dp, dp, dp]
        L.orc_advance.restype = C.c_int

    # ---- noise -----------------------------------------------------------
    def philox(self, ctr, key):
        c = (C.c_uint32 * 4)(*[int(v) & 0xFFFFFFFF for v in ctr])
        k = (C.c_uint32 * 2)(*[int(v) & 0xFFFFFFFF for v in key])
        o = (C.c_uint32 * 4)()
        self.lib.orc_philox4x32_10(c, k, o)
        return [int(v) for v in o]

    def ln_u24(self, w):
        return float(np.float32(self.lib.orc_ln_u24(int(w))))

    def sincos_2pi_u(self, w):
        s, c = C.c_float(), C.c_float()
        self.lib.orc_sincos_2pi_u(int(w), C.byref(s), C.byref(c))
        return np.float32(s.value), np.float32(c.value)

    def normal4(self, w):
        ww = (C.c_uint32 * 4)(*[int(v) & 0xFFFFFFFF for v in w])
        z = (C.c_float * 4)()
        self.lib.orc_normal4(ww, z)
        return np.array(z, dtype=np.float32)

    def normal4_batch(self, words):
        """orc_normal4 over [n][4] Philox words: z [n][4] (float32)."""
        w = np.ascontiguousarray(np.asarray(words, dtype=np.uint32).reshape(-1, 4))
        z = np.zeros(w.shape, dtype=np.float32)
        self.lib.orc_normal4_batch(w.ctypes.data_as(C.POINTER(C.c_uint32)), w.shape[0],
                                   z.ctypes.data_as(C.POINTER(C.c_float)))
        return z

    def sample(self, cfg, mu_shift, var, cur_idx, it, robot, k):
        c = make_config(cfg)
        D = 12 * cfg["knots"]
        th = np.zeros(D)
        z = np.zeros(D, dtype=np.float32)
        idx = C.c_int32()
        self.lib.orc_sample(C.byref(c), _dp(_f64(mu_shift, D)), _dp(_f64(var, D)), int(cur_idx),
                            int(it), int(robot), int(k), _dp(th),
                            z.ctypes.data_as(C.POINTER(C.c_float)), C.byref(idx))
        return th, z, idx.value

    def warm_shift(self, cfg, mu):
        c = make_config(cfg)
        D = 12 * cfg["knots"]
        out = np.zeros(D)
        self.lib.orc_warm_shift(C.byref(c), _dp(_f64(mu, D)), _dp(out))
        return out

    # ---- gait ------------------------------------------------------------
    def phase_inc(self, f, dt):
        return int(self.lib.orc_phase_inc(float(f), float(dt)))

    def stance_threshold(self, duty):
        return int(self.lib.orc_stance_threshold(float(duty)))

    def contact_sequence(self, cfg, phase0, f):
        c = make_config(cfg)
        d = np.zeros((cfg["horizon"], 4), dtype=np.int32)
        self.lib.orc_contact_sequence(C.byref(c), int(phase0) & 0xFFFFFFFF, float(f),
                                      d.ctypes.data_as(C.POINTER(C.c_int32)))
        return d

    # ---- spline / cone ---------------------------------------------------
    def spline_eval(self, knots, a_num, a_den):
        kn = _f64(knots)
        o = C.c_double()
        self.lib.orc_spline_eval(len(kn), _dp(kn), int(a_num), int(a_den), C.byref(o))
        return o.value

    def spline_step(self, cfg, theta, j):
        c = make_config(cfg)
        g = np.zeros(12)
        self.lib.orc_spline_step(C.byref(c), _dp(_f64(theta, 12 * cfg["knots"])), int(j), _dp(g))
        return g

    def cone(self, cfg, raw):
        c = make_config(cfg)
        o = np.zeros(3)
        pen = C.c_double()
        self.lib.orc_cone(C.byref(c), _dp(_f64(raw, 3)), _dp(o), C.byref(pen))
        return o, pen.value

    # ---- dynamics --------------------------------------------------------
    def dynamics(self, cfg, x, gamma, stance, feet):
        c = make_config(cfg)
        xd = np.zeros(12)
        st = np.ascontiguousarray(np.asarray(stance, dtype=np.int32))
        self.lib.orc_dynamics(C.byref(c), _dp(_f64(x, 12)), _dp(_f64(gamma, 12)),
                              st.ctypes.data_as(C.POINTER(C.c_int32)), _dp(_f64(feet, 12)), _dp(xd))
        return xd

    def rk4(self, cfg, x, gamma, stance, feet, h):
        c = make_config(cfg)
        xn = np.zeros(12)
        st = np.ascontiguousarray(np.asarray(stance, dtype=np.int32))
        self.lib.orc_rk4(C.byref(c), _dp(_f64(x, 12)), _dp(_f64(gamma, 12)),
                         st.ctypes.data_as(C.POINTER(C.c_int32)), _dp(_f64(feet, 12)), float(h), _dp(xn))
        return xn

    def rollout(self, cfg, x0, phase0, feet_cur, feet_next, xref, theta, fidx, traj=False):
        c = make_config(cfg)
        H = cfg["horizon"]
        tr = np.zeros((H + 1, 12)) if traj else None
        J = self.lib.orc_rollout(C.byref(c), _dp(_f64(x0, 12)), int(phase0) & 0xFFFFFFFF,
                                 _dp(_f64(feet_cur, 12)), _dp(_f64(feet_next, 12)),
                                 _dp(_f64(xref, H * 12)), _dp(_f64(theta, 12 * cfg["knots"])),
                                 int(fidx), _dp(tr) if traj else None)
        return (J, tr) if traj else J

    def _count_lib(self):
        if not hasattr(self, "_cnt"):
            self._cnt = C.CDLL(_CNT_LIB)
            self._cnt.orc_count_rollout.argtypes = [
                C.POINTER(OrcConfig), C.POINTER(C.c_double), C.c_uint32, C.POINTER(C.c_double),
                C.POINTER(C.c_double), C.POINTER(C.c_double), C.POINTER(C.c_double), C.c_int32,
                C.POINTER(C.c_uint64)]
            self._cnt.orc_count_rollout.restype = C.c_double
            self._cnt.orc_count_sample.argtypes = [
                C.POINTER(OrcConfig), C.POINTER(C.c_double), C.POINTER(C.c_double), C.c_int32, C.c_uint32,
                C.c_uint32, C.c_int64, C.POINTER(C.c_double), C.POINTER(C.c_uint64)]
            self._cnt.orc_count_mppi.argtypes = [C.c_int64, C.c_int32, C.POINTER(C.c_double),
                                                 C.POINTER(C.c_double), C.c_double, C.POINTER(C.c_double),
                                                 C.POINTER(C.c_uint64)]
            self._cnt.orc_count_mppi.restype = C.c_int
        return self._cnt

    def count_rollout(self, cfg, x0, phase0, feet_cur, feet_next, xref, theta, fidx):
        """Op-counting mode (opcount.cpp): (J, FLOPs, transcendentals, compares) of one
        orc_rollout call, counted on the sample-dependent values."""
        L = self._count_lib()
        c = make_config(cfg)
        H = cfg["horizon"]
        n = (C.c_uint64 * 3)()
        J = L.orc_count_rollout(C.byref(c), _dp(_f64(x0, 12)), int(phase0) & 0xFFFFFFFF,
                                        _dp(_f64(feet_cur, 12)), _dp(_f64(feet_next, 12)),
                                        _dp(_f64(xref, H * 12)), _dp(_f64(theta, 12 * cfg["knots"])),
                                        int(fidx), n)
        return J, int(n[0]), int(n[1]), int(n[2])

    def count_sample(self, cfg, mu_shift, var, cur_idx, it, robot, k):
        """Op-counting mode of orc_sample: (theta2, FLOPs, transcendentals, compares)."""
        L = self._count_lib()
        c = make_config(cfg)
        th = np.zeros(12 * cfg["knots"])
        n = (C.c_uint64 * 3)()
        L.orc_count_sample(C.byref(c), _dp(_f64(mu_shift)), _dp(_f64(var)), int(cur_idx), int(it) & 0xFFFFFFFF,
                           int(robot), int(k), _dp(th), n)
        return th, int(n[0]), int(n[1]), int(n[2])

    def count_mppi(self, J, theta, lam):
        """Op-counting mode of orc_mppi: (mu_new, FLOPs, transcendentals, compares)."""
        L = self._count_lib()
        J = _f64(J)
        th = _f64(theta)
        D = th.shape[1]
        mu = np.zeros(D)
        n = (C.c_uint64 * 3)()
        L.orc_count_mppi(len(J), D, _dp(J), _dp(th), float(lam), _dp(mu), n)
        return mu, int(n[0]), int(n[1]), int(n[2])

    # ---- updates ---------------------------------------------------------
    def mppi(self, J, theta, lam):
        J = _f64(J)
        th = _f64(theta)
        K = J.size
        D = th.size // max(K, 1)
        mu = np.zeros(D)
        dg = OrcDiag()
        rc = self.lib.orc_mppi(K, D, _dp(J), _dp(th), float(lam), _dp(mu), C.byref(dg))
        return rc, mu, dg

    def cem_select(self, J, K_e):
        J = _f64(J)
        e = np.zeros(int(K_e), dtype=np.int64)
        rc = self.lib.orc_cem_select(J.size, _dp(J), int(K_e), e.ctypes.data_as(C.POINTER(C.c_int64)))
        assert rc == 0, rc
        return e

    def cem_update(self, J, theta, K_e, var_floor, update_var, var_in):
        J = _f64(J)
        th = _f64(theta)
        K = J.size
        D = th.size // K
        mu = np.zeros(D)
        var = _f64(var_in, D).copy()
        e = np.zeros(int(K_e), dtype=np.int64)
        dg = OrcDiag()
        rc = self.lib.orc_cem_update(K, D, _dp(J), _dp(th), int(K_e), _dp(_f64(var_floor, D)),
                                     int(update_var), _dp(mu), _dp(var),
                                     e.ctypes.data_as(C.POINTER(C.c_int64)), C.byref(dg))
        return rc, mu, var, e, dg

    # ---- whole iteration -------------------------------------------------
    def step(self, cfg, robot, inp, state, keep=True):
        """One Alg. 5 iteration.  ``state`` = dict(mean, var, freq_idx, iter); updated in place."""
        c = make_config(cfg)
        K, D, H = cfg["n_samples"], 12 * cfg["knots"], cfg["horizon"]
        st = OrcState()
        st.mean[:D] = list(np.asarray(state["mean"], dtype=np.float64))
        st.var[:D] = list(np.asarray(state["var"], dtype=np.float64))
        st.freq_idx = int(state["freq_idx"])
        st.iter = int(state["iter"])
        if cfg.get("full_cov", 0):
            st.chol[:D * D] = [float(v) for v in np.asarray(state["chol"], dtype=np.float64).reshape(D * D)]
        out = OrcOutput()
        J = np.zeros(K) if keep else None
        fidx = np.zeros(K, dtype=np.int32) if keep else None
        theta = np.zeros((K, D)) if keep else None
        z = np.zeros((K, D), dtype=np.float32) if keep else None
        ke = 1 if cfg["mode"] == "naive" else (cfg["n_elite"] if cfg["mode"] == "cem" else 0)
        elite = np.zeros(max(ke, 1), dtype=np.int64) if keep and ke else None
        rc = self.lib.orc_step(
            C.byref(c), int(robot), _dp(_f64(inp["x0"], 12)), int(inp["phase"]) & 0xFFFFFFFF,
            _dp(_f64(inp["feet_cur"], 12)), _dp(_f64(inp["feet_next"], 12)),
            _dp(_f64(inp["xref"], H * 12)), C.byref(st), C.byref(out),
            _dp(J) if keep else None, fidx.ctypes.data_as(C.POINTER(C.c_int32)) if keep else None,
            _dp(theta) if keep else None, z.ctypes.data_as(C.POINTER(C.c_float)) if keep else None,
            elite.ctypes.data_as(C.POINTER(C.c_int64)) if elite is not None else None)
        state["mean"] = np.array(st.mean[:D])
        state["var"] = np.array(st.var[:D])
        state["freq_idx"] = st.freq_idx
        state["iter"] = st.iter
        if cfg.get("full_cov", 0):
            state["chol"] = np.array(st.chol[:D * D]).reshape(D, D)
        dg = out.diag
        return StepResult(status=rc, mean=state["mean"].copy(), var=state["var"].copy(),
                          freq_idx=out.freq_idx, freq_hz=out.freq_hz, u0=np.array(out.u0),
                          contact0=np.array(out.contact0), j_min=dg.j_min, j_mean=dg.j_mean,
                          omega=dg.omega, ess=dg.ess, n_diverged=dg.n_diverged, argmin=dg.argmin,
                          J=J, fidx=fidx, theta=theta, z=z, elite=elite)

    # ---- closed loop (L36-L40) -------------------------------
    def foothold(self, p_hip, v_c, v_d, p_cz, t_st, g):
        out = np.zeros(3)
        self.lib.orc_foothold(_dp(_f64(p_hip, 3)), _dp(_f64(v_c, 3)), _dp(_f64(v_d, 3)), float(p_cz),
                              float(t_st), float(g), _dp(out))
        return out

    def plant_dynamics(self, cfg, x, gamma, stance, feet, wrench):
        xd = np.zeros(12)
        st = np.asarray(stance, dtype=np.int32)
        self.lib.orc_plant_dynamics(C.byref(make_config(cfg)), _dp(_f64(x, 12)), _dp(_f64(gamma, 12)),
                                    st.ctypes.data_as(C.POINTER(C.c_int32)), _dp(_f64(feet, 12)),
                                    _dp(_f64(wrench, 6)), _dp(xd))
        return xd

    def plant_step(self, cfg, x, gamma, stance, feet, wrench, h):
        xn = np.zeros(12)
        st = np.asarray(stance, dtype=np.int32)
        self.lib.orc_plant_step(C.byref(make_config(cfg)), _dp(_f64(x, 12)), _dp(_f64(gamma, 12)),
                                st.ctypes.data_as(C.POINTER(C.c_int32)), _dp(_f64(feet, 12)),
                                _dp(_f64(wrench, 6)), float(h), _dp(xn))
        return xn

    def reference(self, cfg, h_nom, x, v_d, yaw_rate):
        xr = np.zeros((cfg["horizon"], 12))
        self.lib.orc_reference(C.byref(make_config(cfg)), float(h_nom), _dp(_f64(x, 12)), _dp(_f64(v_d, 3)),
                               float(yaw_rate), _dp(xr))
        return xr

    def advance(self, cfg, lc, inp, u0, contact0, freq_idx, v_d, yaw_rate=0.0, wrench=None):
        """One closed-loop advance of one robot: plant, fall flag, phase, footholds, reference."""
        x = np.zeros(12)
        ph = C.c_uint32(0)
        fc, fn = np.zeros(12), np.zeros(12)
        xr = np.zeros((cfg["horizon"], 12))
        ct = np.asarray(contact0, dtype=np.int32)
        w = np.zeros(6) if wrench is None else _f64(wrench, 6)
        fallen = self.lib.orc_advance(
            C.byref(make_config(cfg)), C.byref(make_loop_config(lc)), _dp(_f64(inp["x0"], 12)),
            int(inp["phase"]) & 0xFFFFFFFF, _dp(_f64(inp["feet_cur"], 12)), _dp(_f64(inp["feet_next"], 12)),
            _dp(_f64(u0, 12)), ct.ctypes.data_as(C.POINTER(C.c_int32)), int(freq_idx), _dp(_f64(v_d, 3)),
            float(yaw_rate), _dp(w), _dp(x), C.byref(ph), _dp(fc), _dp(fn), _dp(xr))
        return AdvanceResult(fallen=int(fallen), x0=x, phase=int(ph.value), feet_cur=fc, feet_next=fn, xref=xr)

    # ---- full covariance (f3; L42) ---------------------------------------
    def cholesky(self, Cm):
        Cm = _f64(Cm)
        D = int(round(np.sqrt(Cm.size)))
        Lm = np.zeros((D, D))
        rc = self.lib.orc_cholesky(D, _dp(Cm), _dp(Lm))
        return rc, Lm

    def sample_full(self, cfg, mu_shift, Lm, cur_idx, it, robot, k):
        D = 12 * cfg["knots"]
        th = np.zeros(D)
        z = np.zeros(D, dtype=np.float32)
        idx = C.c_int32(0)
        self.lib.orc_sample_full(C.byref(make_config(cfg)), _dp(_f64(mu_shift, D)), _dp(_f64(Lm, D * D)),
                                 int(cur_idx), int(it) & 0xFFFFFFFF, int(robot), int(k), _dp(th),
                                 z.ctypes.data_as(C.POINTER(C.c_float)), C.byref(idx))
        return th, z, idx.value

    def cem_update_full(self, J, theta, K_e, var_floor):
        J = _f64(J)
        th = _f64(theta)
        K = J.size
        D = th.size // K
        mu = np.zeros(D)
        Cn, Ln = np.zeros((D, D)), np.zeros((D, D))
        e = np.zeros(int(K_e), dtype=np.int64)
        dg = OrcDiag()
        rc = self.lib.orc_cem_update_full(K, D, _dp(J), _dp(th), int(K_e), _dp(_f64(var_floor, D)), _dp(mu),
                                          _dp(Cn), _dp(Ln), e.ctypes.data_as(C.POINTER(C.c_int64)), C.byref(dg))
        return rc, mu, Cn, Ln, e, dg
