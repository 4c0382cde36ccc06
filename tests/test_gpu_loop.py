"""GPU parity of the closed loop around the iteration (DESIGN L36-L40):
sbs_advance against the oracle's orc_advance on the same inputs, the graph-
captured sbs_run_loop against step-by-step calls, and whole closed-loop
iterations against the oracle along the GPU's own trajectory.

  plant state, footholds, reference ..... <= 1e-5 max(|ref|, 1)  (binary32 RK4 of one period)
  phase, touchdown copies, fall flag .... bitwise / exact
"""
import ctypes as C

import numpy as np
import pytest

from paper_2403_11383_b200 import workloads as W

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def B():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2403_11383_b200 import binding, build
    build.build()
    binding.load_library()
    return binding


def _dev_bytes(arr):
    import torch
    return torch.from_numpy(np.frombuffer(bytes(arr), dtype=np.uint8).copy()).cuda()


def _inputs_of(B, d_in, R):
    raw = d_in.cpu().numpy().tobytes()
    n = C.sizeof(B.sbs_input)
    out = []
    for r in range(R):
        s = B.sbs_input.from_buffer_copy(raw[r * n:(r + 1) * n])
        out.append(dict(x0=np.array(s.x0, dtype=np.float64), phase=int(s.phase_q32),
                        feet_cur=np.array(s.feet_cur, dtype=np.float64),
                        feet_next=np.array(s.feet_next, dtype=np.float64)))
    return out


def _outputs_of(B, d_out, R, D):
    raw = d_out.cpu().numpy().tobytes()
    n = C.sizeof(B.sbs_output)
    return [B.output_dict(B.sbs_output.from_buffer_copy(raw[r * n:(r + 1) * n]), D) for r in range(R)]


def _close(a, b, rel=1e-5):
    a, b = np.asarray(a, dtype=np.float64), np.asarray(b, dtype=np.float64)
    return np.max(np.abs(a - b)) <= rel * max(1.0, float(np.max(np.abs(b))))


def _commands(R, seed=7):
    rng = np.random.default_rng(seed)
    cmd = np.zeros((R, 4), dtype=np.float32)
    cmd[:, :2] = rng.uniform(-0.5, 0.5, size=(R, 2))
    cmd[:, 3] = rng.uniform(-0.3, 0.3, size=R)
    return cmd


def test_advance_matches_oracle(B, orc):
    import torch
    R = 64
    cfg, inputs = W.config5(R=R, M=256)
    inputs[5]["x0"] = inputs[5]["x0"].copy()
    inputs[5]["x0"][2] = 0.10                                      # falls this period (L40)
    inputs[9]["x0"] = inputs[9]["x0"].copy()
    inputs[9]["x0"][6] = 0.9                                       # tilted past the fall angle
    inputs[0]["phase"] = W.q32(0.499)                              # FR/RL land this period
    inputs[1]["phase"] = W.q32(0.999)                              # FL/RR land this period
    lc = W.loop_config()
    c = B.Controller(cfg)
    for r, inp in enumerate(inputs):
        c.set_reference(r, inp["xref"])
    d_in = _dev_bytes(B.make_inputs(inputs))
    d_out = torch.zeros(R * C.sizeof(B.sbs_output), dtype=torch.uint8, device="cuda")
    cmd = _commands(R)
    d_cmd = torch.from_numpy(cmd).cuda()
    wrench = np.random.default_rng(1).uniform(-20, 20, size=(R, 6)).astype(np.float32)
    d_w = torch.from_numpy(wrench).cuda()
    d_fallen = torch.zeros(R, dtype=torch.int32, device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    c.step_device(d_in.data_ptr(), d_out.data_ptr(), s)
    before = _inputs_of(B, d_in, R)
    outs = _outputs_of(B, d_out, R, 48)
    c.advance(d_in.data_ptr(), d_out.data_ptr(), d_cmd.data_ptr(), d_w.data_ptr(), d_fallen.data_ptr(), lc, s)
    torch.cuda.synchronize()
    after = _inputs_of(B, d_in, R)
    fallen = d_fallen.cpu().numpy()
    n_land = 0
    for r in range(R):
        o = outs[r]
        ro = orc.advance(cfg, lc, before[r], o["u0"], o["contact0"], o["freq_idx"], cmd[r, :3], float(cmd[r, 3]),
                         wrench[r])
        assert after[r]["phase"] == ro.phase
        assert fallen[r] == ro.fallen, r
        assert _close(after[r]["x0"], ro.x0), (r, after[r]["x0"] - ro.x0)
        np.testing.assert_array_equal(after[r]["feet_cur"], ro.feet_cur.astype(np.float32))   # copies only
        assert _close(after[r]["feet_next"], ro.feet_next)
        assert _close(c.get_reference(r), ro.xref)
        n_land += int(not np.array_equal(after[r]["feet_cur"], before[r]["feet_cur"]))
    assert fallen[5] == 1 and fallen[9] == 1 and fallen.sum() == 2
    assert n_land > 0                                              # some legs touched down this period


def test_fallen_robot_is_frozen(B):
    import torch
    cfg, inputs = W.config5(R=4, M=128)
    lc = W.loop_config()
    c = B.Controller(cfg)
    for r, inp in enumerate(inputs):
        c.set_reference(r, inp["xref"])
    d_in = _dev_bytes(B.make_inputs(inputs))
    d_out = torch.zeros(4 * C.sizeof(B.sbs_output), dtype=torch.uint8, device="cuda")
    d_fallen = torch.tensor([0, 1, 0, 0], dtype=torch.int32, device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    c.step_device(d_in.data_ptr(), d_out.data_ptr(), s)
    before = d_in.clone()
    c.advance(d_in.data_ptr(), d_out.data_ptr(), 0, 0, d_fallen.data_ptr(), lc, s)
    n = C.sizeof(B.sbs_input)
    a, b = d_in.cpu().numpy(), before.cpu().numpy()
    assert np.array_equal(a[n:2 * n], b[n:2 * n])                  # robot 1 frozen
    assert not np.array_equal(a[:n], b[:n])                        # robot 0 advanced


@pytest.mark.parametrize("mode", ["mppi", "naive", "cem", "cem-fc", "mppi-dyn"])
def test_run_loop_equals_stepwise_calls(B, mode):
    """sbs_run_loop (captured iterations replayed, iteration counter in device memory) is
    bitwise the same as n x (sbs_step_device + sbs_advance); mppi-dyn: one robot at
    K = 2^18, where the rollout schedules its tiles dynamically inside the graph."""
    import torch
    R, n = 3, 25
    fc = mode == "cem-fc"
    dyn = mode == "mppi-dyn"
    mode = "cem" if fc else ("mppi" if dyn else mode)
    if dyn:
        R, n = 1, 10
    cfg = W.base_config(n_samples=(1 << 18) if dyn else 2000, n_elite=200 if mode == "cem" else 1, mode=mode,
                        n_robots=R, gait_adapt=0 if mode == "mppi" else 1, full_cov=1 if fc else 0)
    inputs = [W.robot_input(cfg, r, cmd=(0.3, 0.1 * r, 0), phase=W.q32(0.1 * r)) for r in range(R)]
    lc = W.loop_config()
    cmd = torch.from_numpy(_commands(R)).cuda()
    wrench = torch.from_numpy(np.random.default_rng(2).uniform(-20, 20, size=(n, R, 6)).astype(np.float32)).cuda()
    s = torch.cuda.current_stream().cuda_stream
    res = []
    for use_loop in (True, False):
        c = B.Controller(cfg)
        for r, inp in enumerate(inputs):
            c.set_reference(r, inp["xref"])
        d_in = _dev_bytes(B.make_inputs(inputs))
        d_out = torch.zeros(R * C.sizeof(B.sbs_output), dtype=torch.uint8, device="cuda")
        fallen = torch.zeros(R, dtype=torch.int32, device="cuda")
        trace = torch.zeros((n, R, B.SBS_TRACE_FLOATS), dtype=torch.float32, device="cuda")
        if use_loop:
            c.run_loop(n, d_in.data_ptr(), d_out.data_ptr(), cmd.data_ptr(), wrench.data_ptr(), fallen.data_ptr(),
                       trace.data_ptr(), lc, s)
        else:
            for i in range(n):
                c.step_device(d_in.data_ptr(), d_out.data_ptr(), s)
                c.advance(d_in.data_ptr(), d_out.data_ptr(), cmd.data_ptr(), wrench[i].data_ptr(), fallen.data_ptr(),
                          lc, s)
                o = _outputs_of(B, d_out, R, 48)
                x = _inputs_of(B, d_in, R)
                for r in range(R):
                    trace[i, r, :12] = torch.tensor(x[r]["x0"], dtype=torch.float32)
                    trace[i, r, 12] = o[r]["freq_hz"]
                    trace[i, r, 13] = o[r]["j_min"]
                    trace[i, r, 15] = o[r]["status"]
        torch.cuda.synchronize()
        assert c.iter == n
        m = [c.get_distribution(r)[0] for r in range(R)]
        t = trace.cpu().numpy()
        t[:, :, 14] = 0
        res.append((d_in.cpu().numpy(), d_out.cpu().numpy(), np.array(m), t))
    for a, b in zip(res[0], res[1]):
        np.testing.assert_array_equal(a, b)


def test_closed_loop_iterations_match_oracle_along_the_gpu_trajectory(B, orc):
    """Ten closed-loop iterations (MPPI, gait adaptation off): before each one the
    GPU's inputs, reference and distribution are handed to the oracle, which runs the
    same iteration (sampling, rollouts, update) and the same advance."""
    import torch
    R, n = 2, 10
    cfg = W.base_config(n_samples=256, mode="mppi", n_robots=R)
    inputs = [W.robot_input(cfg, r, cmd=(0.4, -0.1, 0), phase=W.q32(0.2 + 0.3 * r)) for r in range(R)]
    lc = W.loop_config()
    cmd_np = np.tile(np.array([0.4, -0.1, 0.0, 0.1], dtype=np.float32), (R, 1))
    cmd = torch.from_numpy(cmd_np).cuda()
    wrench_np = np.random.default_rng(4).uniform(-10, 10, size=(n, R, 6)).astype(np.float32)
    c = B.Controller(cfg)
    for r, inp in enumerate(inputs):
        c.set_reference(r, inp["xref"])
    d_in = _dev_bytes(B.make_inputs(inputs))
    d_out = torch.zeros(R * C.sizeof(B.sbs_output), dtype=torch.uint8, device="cuda")
    fallen = torch.zeros(R, dtype=torch.int32, device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    for i in range(n):
        gin = _inputs_of(B, d_in, R)
        states = []
        for r in range(R):
            m, v, f = c.get_distribution(r)
            states.append(dict(mean=m.astype(np.float64), var=v.astype(np.float64), freq_idx=f, iter=c.iter))
            gin[r]["xref"] = c.get_reference(r).astype(np.float64)
        c.step_device(d_in.data_ptr(), d_out.data_ptr(), s)
        w = torch.from_numpy(wrench_np[i]).cuda()
        c.advance(d_in.data_ptr(), d_out.data_ptr(), cmd.data_ptr(), w.data_ptr(), fallen.data_ptr(), lc, s)
        torch.cuda.synchronize()
        outs = _outputs_of(B, d_out, R, 48)
        gnext = _inputs_of(B, d_in, R)
        for r in range(R):
            ro = orc.step(cfg, r, gin[r], states[r], keep=False)
            o = outs[r]
            assert o["status"] == ro.status and o["freq_idx"] == ro.freq_idx
            np.testing.assert_array_equal(o["contact0"], ro.contact0)
            assert np.max(np.abs(o["mean"] - ro.mean)) <= 1e-4 * max(np.max(np.abs(ro.mean)), 1.0)
            assert np.max(np.abs(o["u0"] - ro.u0)) <= 1e-4 * max(np.max(np.abs(ro.u0)), 1.0)
            ra = orc.advance(cfg, lc, gin[r], o["u0"], o["contact0"], o["freq_idx"], cmd_np[r, :3],
                             float(cmd_np[r, 3]), wrench_np[i, r])
            assert gnext[r]["phase"] == ra.phase
            assert _close(gnext[r]["x0"], ra.x0) and _close(gnext[r]["feet_next"], ra.feet_next)
            np.testing.assert_array_equal(gnext[r]["feet_cur"], ra.feet_cur.astype(np.float32))
            assert _close(c.get_reference(r), ra.xref)
    assert c.iter == n and int(fallen.sum()) == 0


def test_inner_iterations_match_oracle(B, orc):
    """n_inner = 3 SBS iterations per control step (Alg. 1 "multiple times"; L34):
    the first with the warm shift, the others refining the same distribution at the same
    x0 with fresh noise (iteration counter + 1 each), then one advance."""
    import torch
    R, inner = 2, 3
    cfg = W.base_config(n_samples=300, mode="mppi", n_robots=R)
    inputs = [W.robot_input(cfg, r, cmd=(0.2, 0.1, 0), phase=W.q32(0.3 * r)) for r in range(R)]
    lc = dict(W.loop_config(), n_inner=inner)
    cmd_np = np.tile(np.array([0.2, 0.1, 0.0, 0.0], dtype=np.float32), (R, 1))
    c = B.Controller(cfg)
    for r, inp in enumerate(inputs):
        c.set_reference(r, inp["xref"])
    d_in = _dev_bytes(B.make_inputs(inputs))
    d_out = torch.zeros(R * C.sizeof(B.sbs_output), dtype=torch.uint8, device="cuda")
    cmd = torch.from_numpy(cmd_np).cuda()
    s = torch.cuda.current_stream().cuda_stream
    for step in range(3):
        gin = _inputs_of(B, d_in, R)
        states = []
        for r in range(R):
            m, v, f = c.get_distribution(r)
            states.append(dict(mean=m.astype(np.float64), var=v.astype(np.float64), freq_idx=f, iter=c.iter))
            gin[r]["xref"] = c.get_reference(r).astype(np.float64)
        c.run_loop(1, d_in.data_ptr(), d_out.data_ptr(), cmd.data_ptr(), 0, 0, 0, lc, s)
        torch.cuda.synchronize()
        assert c.iter == inner * (step + 1)
        outs = _outputs_of(B, d_out, R, 48)
        gnext = _inputs_of(B, d_in, R)
        for r in range(R):
            st = states[r]
            for k in range(inner):
                ro = orc.step(cfg if k == 0 else dict(cfg, warm_shift=0), r, gin[r], st, keep=False)
            o = outs[r]
            assert np.max(np.abs(o["mean"] - ro.mean)) <= 1e-4 * max(np.max(np.abs(ro.mean)), 1.0)
            assert np.max(np.abs(o["u0"] - ro.u0)) <= 1e-4 * max(np.max(np.abs(ro.u0)), 1.0)
            ra = orc.advance(cfg, lc, gin[r], o["u0"], o["contact0"], o["freq_idx"], cmd_np[r, :3], 0.0)
            assert gnext[r]["phase"] == ra.phase
            assert _close(gnext[r]["x0"], ra.x0)
