"""Thin ctypes binding of the C ABI in include/sbs.h (libsbs.so).

Argument marshalling only: every step of the MPC iteration runs in the CUDA
kernels behind the library.  Importing works without a GPU (the library is
cross-compiled); there is no CPU fallback -- calls fail loudly when the
library is missing or the device is absent.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SBS_LIB_PATH", os.path.join(HERE, "libsbs.so"))  # override: experiments only

SBS_MAX_KNOTS = 8
SBS_MAX_D = 12 * SBS_MAX_KNOTS
SBS_MAX_FREQ = 8
SBS_MAX_HORIZON = 64
MODES = {"mppi": 0, "cem": 1, "naive": 2}
STATUS = {0: "SBS_OK", 1: "SBS_WARN_ALL_DIVERGED", -1: "SBS_ERR_INVALID_ARG", -2: "SBS_ERR_SINGULAR",
          -3: "SBS_ERR_NONFINITE", -4: "SBS_ERR_STATE", -5: "SBS_ERR_CUDA", -6: "SBS_ERR_NCCL", -7: "SBS_ERR_OOM"}
KERNELS = ["rollout", "reduce", "select", "elite", "advance"]


class sbs_config(C.Structure):
    _fields_ = [
        ("mass", C.c_float), ("inertia", C.c_float * 9), ("gravity", C.c_float * 3),
        ("mu", C.c_float), ("fz_min", C.c_float), ("fz_max", C.c_float),
        ("horizon", C.c_int32), ("knots", C.c_int32), ("dt", C.c_float),
        ("duty_factor", C.c_float), ("phase_offset", C.c_float * 4),
        ("n_freq", C.c_int32), ("gait_adapt", C.c_int32), ("freq_hz", C.c_float * SBS_MAX_FREQ),
        ("Q", C.c_float * 12), ("R", C.c_float * 12), ("rho", C.c_float), ("f_nominal", C.c_float),
        ("w_fc", C.c_float),
        ("mode", C.c_int32), ("elite_preserve", C.c_int32), ("n_samples", C.c_int64), ("n_elite", C.c_int64),
        ("lambda_", C.c_float), ("sigma", C.c_float * 3), ("sigma_min_frac", C.c_float),
        ("warm_shift", C.c_int32), ("seed", C.c_uint64),
        ("n_robots", C.c_int32), ("robot_offset", C.c_int32), ("device", C.c_int32),
        ("rank", C.c_int32), ("world", C.c_int32), ("nccl_id", C.c_uint8 * 128),
        ("n_sigma_groups", C.c_int32), ("sigma_scale", C.c_float * 8), ("full_cov", C.c_int32),
    ]


class sbs_input(C.Structure):
    _fields_ = [("x0", C.c_float * 12), ("phase_q32", C.c_uint32), ("feet_cur", C.c_float * 12),
                ("feet_next", C.c_float * 12), ("_pad", C.c_uint32 * 3)]


class sbs_output(C.Structure):
    _fields_ = [("u0", C.c_float * 12), ("contact0", C.c_uint8 * 4), ("freq_idx", C.c_int32),
                ("freq_hz", C.c_float), ("status", C.c_int32), ("iter", C.c_uint32), ("j_min", C.c_float),
                ("j_mean", C.c_float), ("omega", C.c_float), ("ess", C.c_float), ("n_diverged", C.c_int32),
                ("device_us", C.c_float), ("mean", C.c_float * SBS_MAX_D), ("var", C.c_float * SBS_MAX_D)]


class sbs_loop_config(C.Structure):
    _fields_ = [("hip", C.c_float * 12), ("h_nom", C.c_float), ("fall_angle", C.c_float),
                ("fall_height", C.c_float), ("n_inner", C.c_int32)]


class sbs_command(C.Structure):
    _fields_ = [("v", C.c_float * 3), ("yaw_rate", C.c_float)]


SBS_TRACE_FLOATS = 16


def make_loop_config(lc: dict) -> sbs_loop_config:
    o = sbs_loop_config()
    o.hip[:] = [float(v) for v in np.asarray(lc["hip"], dtype=np.float64).reshape(12)]
    o.h_nom, o.fall_angle, o.fall_height = float(lc["h_nom"]), float(lc["fall_angle"]), float(lc["fall_height"])
    o.n_inner = int(lc.get("n_inner", 1))
    return o


class SBSError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status


_lib = None


def load_library(path: str = LIB_PATH):
    """Load libsbs.so; raise if it is missing (no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError(f"{path} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`")
    L = C.CDLL(path)
    P, vp = C.POINTER, C.c_void_p
    ctxp = vp
    sig = {
        "sbs_version": ([], C.c_int),
        "sbs_sizeof_config": ([], C.c_uint64),
        "sbs_sizeof_input": ([], C.c_uint64),
        "sbs_sizeof_output": ([], C.c_uint64),
        "sbs_status_str": ([C.c_int], C.c_char_p),
        "sbs_last_error": ([ctxp], C.c_char_p),
        "sbs_create": ([P(sbs_config), P(ctxp)], C.c_int),
        "sbs_destroy": ([ctxp], None),
        "sbs_set_reference": ([ctxp, C.c_int32, vp], C.c_int),
        "sbs_set_reference_device": ([ctxp, vp, vp], C.c_int),
        "sbs_set_distribution": ([ctxp, C.c_int32, P(C.c_float), P(C.c_float), C.c_int32], C.c_int),
        "sbs_get_distribution": ([ctxp, C.c_int32, P(C.c_float), P(C.c_float), P(C.c_int32)], C.c_int),
        "sbs_get_iter": ([ctxp], C.c_uint32),
        "sbs_set_iter": ([ctxp, C.c_uint32], C.c_int),
        "sbs_step": ([ctxp, P(sbs_input), P(sbs_output)], C.c_int),
        "sbs_step_device": ([ctxp, vp, vp, vp], C.c_int),
        "sbs_get_state": ([ctxp, vp, P(C.c_uint64)], C.c_int),
        "sbs_set_state": ([ctxp, vp, C.c_uint64], C.c_int),
        "sbs_nccl_unique_id": ([P(C.c_uint8)], C.c_int),
        "sbs_debug_samples": ([ctxp, C.c_int32, C.c_int64, C.c_int64, P(C.c_float), P(C.c_float), P(C.c_int32)],
                              C.c_int),
        "sbs_debug_costs": ([ctxp, P(C.c_float)], C.c_int),
        "sbs_debug_elites": ([ctxp, C.c_int32, P(C.c_int64)], C.c_int),
        "sbs_debug_select": ([P(C.c_float), C.c_int64, C.c_int64, P(C.c_int64), C.c_int32], C.c_int),
        "sbs_local_range": ([ctxp, P(C.c_int64), P(C.c_int64)], C.c_int),
        "sbs_debug_noise": ([P(C.c_uint32), C.c_int64, P(C.c_float), C.c_int32], C.c_int),
        "sbs_debug_philox": ([P(C.c_uint32), P(C.c_uint32), C.c_int64, P(C.c_uint32), P(C.c_uint32), C.c_int32],
                             C.c_int),
        "sbs_profile": ([ctxp, C.c_int32], C.c_int),
        "sbs_kernel_times": ([ctxp, P(C.c_double), P(C.c_int64)], C.c_int),
        "sbs_launches_per_step": ([ctxp], C.c_int),
        "sbs_record_floats": ([ctxp], C.c_int),
        "sbs_step_records": ([ctxp, vp, vp, vp], C.c_int),
        "sbs_peer_handle": ([ctxp, P(C.c_uint8), P(vp)], C.c_int),
        "sbs_peer_connect": ([ctxp, P(vp), P(C.c_uint8)], C.c_int),
        "sbs_finish_records": ([ctxp, vp, vp, vp, vp], C.c_int),
        "sbs_set_covariance": ([ctxp, C.c_int32, P(C.c_float)], C.c_int),
        "sbs_get_cholesky": ([ctxp, C.c_int32, P(C.c_float)], C.c_int),
        "sbs_get_reference": ([ctxp, C.c_int32, P(C.c_float)], C.c_int),
        "sbs_advance": ([ctxp, vp, vp, vp, vp, vp, P(sbs_loop_config), vp], C.c_int),
        "sbs_run_loop": ([ctxp, C.c_int32, vp, vp, vp, vp, vp, vp, P(sbs_loop_config), vp], C.c_int),
    }
    for name, (args, res) in sig.items():
        f = getattr(L, name)
        f.argtypes = args
        f.restype = res
    assert L.sbs_sizeof_config() == C.sizeof(sbs_config), "sbs_config layout mismatch"
    assert L.sbs_sizeof_input() == C.sizeof(sbs_input), "sbs_input layout mismatch"
    assert L.sbs_sizeof_output() == C.sizeof(sbs_output), "sbs_output layout mismatch"
    _lib = L
    return L


def _fp(a):
    return a.ctypes.data_as(C.POINTER(C.c_float))


def make_config(cfg: dict, device: int = 0, rank: int = 0, world: int = 1, nccl_id: bytes | None = None,
                robot_offset: int = 0) -> sbs_config:
    c = sbs_config()
    c.mass = cfg["mass"]
    c.inertia[:] = [float(v) for v in np.asarray(cfg["inertia"]).ravel()]
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
    c.n_samples = int(cfg["n_samples"])
    c.n_elite = int(cfg["n_elite"])
    c.lambda_ = cfg["lambda"]
    c.sigma[:] = list(cfg["sigma"])
    c.sigma_min_frac = cfg["sigma_min_frac"]
    c.warm_shift = int(cfg["warm_shift"])
    c.seed = int(cfg["seed"])
    c.n_robots = int(cfg.get("n_robots", 1))
    c.robot_offset = robot_offset
    c.device, c.rank, c.world = device, rank, world
    if nccl_id is not None:
        c.nccl_id[:] = list(nccl_id)
    sc = list(cfg.get("sigma_scale", [1.0]))
    c.n_sigma_groups = len(sc)
    c.sigma_scale[:len(sc)] = [float(v) for v in sc]
    c.full_cov = int(cfg.get("full_cov", 0))
    return c


def make_inputs(inputs: list[dict]):
    arr = (sbs_input * len(inputs))()
    for i, inp in enumerate(inputs):
        arr[i].x0[:] = [float(v) for v in inp["x0"]]
        arr[i].phase_q32 = int(inp["phase"]) & 0xFFFFFFFF
        arr[i].feet_cur[:] = [float(v) for v in inp["feet_cur"]]
        arr[i].feet_next[:] = [float(v) for v in inp["feet_next"]]
    return arr


def output_dict(o: sbs_output, D: int) -> dict:
    return dict(u0=np.array(o.u0, dtype=np.float32), contact0=np.array(o.contact0, dtype=np.int32),
                freq_idx=o.freq_idx, freq_hz=o.freq_hz, status=o.status, iter=o.iter, j_min=o.j_min,
                j_mean=o.j_mean, omega=o.omega, ess=o.ess, n_diverged=o.n_diverged, device_us=o.device_us,
                mean=np.array(o.mean[:D], dtype=np.float32), var=np.array(o.var[:D], dtype=np.float32))


class Controller:
    """One sbs_ctx (R robots).  Methods mirror the C ABI names."""

    def __init__(self, cfg: dict, device: int = 0, rank: int = 0, world: int = 1, nccl_id: bytes | None = None,
                 robot_offset: int = 0):
        self.L = load_library()
        self.cfg = cfg
        self.R = int(cfg.get("n_robots", 1))
        self.D = 12 * cfg["knots"]
        self.H = cfg["horizon"]
        self._c = make_config(cfg, device, rank, world, nccl_id, robot_offset)
        self.ctx = C.c_void_p()
        self._check(self.L.sbs_create(C.byref(self._c), C.byref(self.ctx)), None)

    def _check(self, st, ctx="self"):
        if st < 0:
            msg = self.L.sbs_last_error(self.ctx if ctx == "self" else None)
            raise SBSError(st, (msg or b"").decode())
        return st

    def close(self):
        if self.ctx:
            self.L.sbs_destroy(self.ctx)
            self.ctx = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ---- state --------------------------------------------------------------
    def set_reference(self, robot: int, xref):
        a = xref
        if not (isinstance(a, np.ndarray) and a.dtype == np.float32 and a.flags.c_contiguous and a.size == self.H * 12):
            a = np.ascontiguousarray(np.asarray(xref, dtype=np.float32).reshape(self.H, 12))
        return self._check(self.L.sbs_set_reference(self.ctx, robot, a.ctypes.data))

    def set_reference_device(self, d_ptr: int, stream: int = 0):
        return self._check(self.L.sbs_set_reference_device(self.ctx, C.c_void_p(d_ptr), C.c_void_p(stream)))

    def set_distribution(self, robot: int, mean, var, freq_idx: int):
        m = np.ascontiguousarray(np.asarray(mean, dtype=np.float32))
        v = np.ascontiguousarray(np.asarray(var, dtype=np.float32))
        return self._check(self.L.sbs_set_distribution(self.ctx, robot, _fp(m), _fp(v), int(freq_idx)))

    def get_distribution(self, robot: int):
        m = np.zeros(self.D, dtype=np.float32)
        v = np.zeros(self.D, dtype=np.float32)
        f = C.c_int32()
        self._check(self.L.sbs_get_distribution(self.ctx, robot, _fp(m), _fp(v), C.byref(f)))
        return m, v, f.value

    @property
    def iter(self) -> int:
        return int(self.L.sbs_get_iter(self.ctx))

    @iter.setter
    def iter(self, v: int):
        self._check(self.L.sbs_set_iter(self.ctx, int(v)))

    def get_state(self) -> bytes:
        n = C.c_uint64(0)
        self._check(self.L.sbs_get_state(self.ctx, None, C.byref(n)))
        buf = C.create_string_buffer(n.value)
        self._check(self.L.sbs_get_state(self.ctx, buf, C.byref(n)))
        return buf.raw

    def set_state(self, data: bytes):
        buf = C.create_string_buffer(data, len(data))
        return self._check(self.L.sbs_set_state(self.ctx, buf, len(data)))

    # ---- iteration ----------------------------------------------------------
    def step(self, inputs):
        """sbs_step: host inputs (list of dicts or an sbs_input array), returns (status, [output dict])."""
        arr = inputs if isinstance(inputs, C.Array) else make_inputs(inputs)
        out = (sbs_output * self.R)()
        st = self._check(self.L.sbs_step(self.ctx, arr, out))
        return st, [output_dict(out[r], self.D) for r in range(self.R)]

    def step_raw(self, arr, out):
        """sbs_step with preallocated ctypes arrays (no per-call allocation)."""
        return self._check(self.L.sbs_step(self.ctx, arr, out))

    def step_device(self, d_in: int, d_out: int, stream: int = 0):
        return self._check(self.L.sbs_step_device(self.ctx, C.c_void_p(d_in), C.c_void_p(d_out),
                                                  C.c_void_p(stream)))

    # ---- sample sharding with a caller-driven exchange --------------------------
    def record_floats(self) -> int:
        return int(self.L.sbs_record_floats(self.ctx))

    def step_records(self, d_in: int, d_rec: int, stream: int = 0):
        return self._check(self.L.sbs_step_records(self.ctx, C.c_void_p(d_in), C.c_void_p(d_rec),
                                                   C.c_void_p(stream)))

    # ---- peer-memory exchange (replaces the NCCL all-gather) -----------------------
    def peer_handle(self):
        """(IPC handle bytes, device address) of this rank's exchange buffer."""
        h = (C.c_uint8 * 64)()
        base = C.c_void_p()
        self._check(self.L.sbs_peer_handle(self.ctx, h, C.byref(base)))
        return bytes(h), int(base.value or 0)

    def peer_connect(self, bases=None, handles=None):
        """bases: every rank's device address (same process), or handles: every rank's IPC handle."""
        if bases is None and handles is None:  # disconnect
            return self._check(self.L.sbs_peer_connect(self.ctx, None, None))
        if bases is not None:
            arr = (C.c_void_p * len(bases))(*bases)
            return self._check(self.L.sbs_peer_connect(self.ctx, arr, None))
        blob = b"".join(handles)
        harr = (C.c_uint8 * len(blob)).from_buffer_copy(blob)
        return self._check(self.L.sbs_peer_connect(self.ctx, None, harr))

    def finish_records(self, d_recs: int, d_in: int, d_out: int, stream: int = 0):
        return self._check(self.L.sbs_finish_records(self.ctx, C.c_void_p(d_recs), C.c_void_p(d_in),
                                                     C.c_void_p(d_out), C.c_void_p(stream)))

    # ---- tests / measurement -------------------------------------------------
    def debug_samples(self, robot: int, k0: int, n: int):
        z = np.zeros((n, self.D), dtype=np.float32)
        th = np.zeros((n, self.D), dtype=np.float32)
        f = np.zeros(n, dtype=np.int32)
        self._check(self.L.sbs_debug_samples(self.ctx, robot, k0, n, _fp(z), _fp(th),
                                             f.ctypes.data_as(C.POINTER(C.c_int32))))
        return z, th, f

    def local_range(self):
        a, b = C.c_int64(), C.c_int64()
        self._check(self.L.sbs_local_range(self.ctx, C.byref(a), C.byref(b)))
        return a.value, b.value

    def debug_costs(self):
        _, K = self.local_range()
        J = np.zeros((self.R, K), dtype=np.float32)
        self._check(self.L.sbs_debug_costs(self.ctx, _fp(J)))
        return J

    def debug_elites(self, robot: int = 0):
        ke = 1 if self.cfg["mode"] == "naive" else int(self.cfg["n_elite"])
        idx = np.zeros(ke, dtype=np.int64)
        self._check(self.L.sbs_debug_elites(self.ctx, robot, idx.ctypes.data_as(C.POINTER(C.c_int64))))
        return idx

    def profile(self, enable: bool = True):
        return self._check(self.L.sbs_profile(self.ctx, 1 if enable else 0))

    def kernel_times(self):
        nk = len(KERNELS)
        ms = (C.c_double * nk)()
        n = (C.c_int64 * nk)()
        self._check(self.L.sbs_kernel_times(self.ctx, ms, n))
        return {KERNELS[i]: (ms[i], n[i]) for i in range(nk)}

    def set_covariance(self, robot: int, Cm):
        a = np.ascontiguousarray(np.asarray(Cm, dtype=np.float32).reshape(self.D, self.D))
        return self._check(self.L.sbs_set_covariance(self.ctx, robot, _fp(a)))

    def get_cholesky(self, robot: int = 0):
        Lm = np.zeros((self.D, self.D), dtype=np.float32)
        self._check(self.L.sbs_get_cholesky(self.ctx, robot, _fp(Lm)))
        return Lm

    def get_reference(self, robot: int = 0):
        x = np.zeros((self.H, 12), dtype=np.float32)
        self._check(self.L.sbs_get_reference(self.ctx, robot, _fp(x)))
        return x

    # ---- closed loop: device pointers (ints), 0 for NULL ----
    def advance(self, d_in: int, d_out: int, d_cmd: int, d_wrench: int, d_fallen: int, lc: dict, stream: int = 0):
        lcs = make_loop_config(lc)
        return self._check(self.L.sbs_advance(self.ctx, C.c_void_p(d_in), C.c_void_p(d_out), C.c_void_p(d_cmd or None),
                                              C.c_void_p(d_wrench or None), C.c_void_p(d_fallen or None),
                                              C.byref(lcs), C.c_void_p(stream)))

    def run_loop(self, n_iter: int, d_in: int, d_out: int, d_cmd: int, d_wrench: int, d_fallen: int, d_trace: int,
                 lc: dict, stream: int = 0):
        lcs = make_loop_config(lc)
        return self._check(self.L.sbs_run_loop(self.ctx, int(n_iter), C.c_void_p(d_in), C.c_void_p(d_out),
                                               C.c_void_p(d_cmd or None), C.c_void_p(d_wrench or None),
                                               C.c_void_p(d_fallen or None), C.c_void_p(d_trace or None),
                                               C.byref(lcs), C.c_void_p(stream)))

    def launches_per_step(self) -> int:
        return int(self.L.sbs_launches_per_step(self.ctx))


def debug_select(J, K_e: int, device: int = 0):
    """Stand-alone GPU elite selection of the K_e smallest (J, k); ascending indices."""
    L = load_library()
    J = np.ascontiguousarray(np.asarray(J, dtype=np.float32))
    idx = np.zeros(int(K_e), dtype=np.int64)
    st = L.sbs_debug_select(_fp(J), J.size, int(K_e), idx.ctypes.data_as(C.POINTER(C.c_int64)), device)
    if st < 0:
        raise SBSError(st, (L.sbs_last_error(None) or b"").decode())
    return idx


def debug_noise(words, device: int = 0):
    """The noise recipe on given Philox words [n][4] (uint32) on the GPU: z [n][4] (float32)."""
    L = load_library()
    w = np.ascontiguousarray(np.asarray(words, dtype=np.uint32).reshape(-1, 4))
    z = np.zeros(w.shape, dtype=np.float32)
    st = L.sbs_debug_noise(w.ctypes.data_as(C.POINTER(C.c_uint32)), w.shape[0], _fp(z), device)
    if st < 0:
        raise SBSError(st, (L.sbs_last_error(None) or b"").decode())
    return z


def debug_philox(ctr, key, device: int = 0):
    """Philox4x32-10 on the GPU for counters [n][4] and keys [n][2]: (ours [n][2][4], cuRAND's [n][4])."""
    L = load_library()
    c = np.ascontiguousarray(np.asarray(ctr, dtype=np.uint32).reshape(-1, 4))
    k = np.ascontiguousarray(np.asarray(key, dtype=np.uint32).reshape(-1, 2))
    n = c.shape[0]
    ours = np.zeros((n, 2, 4), dtype=np.uint32)
    cur = np.zeros((n, 4), dtype=np.uint32)
    u32p = C.POINTER(C.c_uint32)
    st = L.sbs_debug_philox(c.ctypes.data_as(u32p), k.ctypes.data_as(u32p), n, ours.ctypes.data_as(u32p),
                            cur.ctypes.data_as(u32p), device)
    if st < 0:
        raise SBSError(st, (L.sbs_last_error(None) or b"").decode())
    return ours, cur


def nccl_unique_id() -> bytes:
    L = load_library()
    buf = (C.c_uint8 * 128)()
    st = L.sbs_nccl_unique_id(buf)
    if st < 0:
        raise SBSError(st, (L.sbs_last_error(None) or b"").decode())
    return bytes(buf)
