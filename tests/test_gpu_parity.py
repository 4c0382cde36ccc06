"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle on the
same seeded inputs.

  noise z, theta1 index, contact flags ......... bitwise
  theta2 ....................................... <= 1e-6 relative (binary32 warm shift)
  costs ........................................ |dJ| <= 1e-4 |J| + 1e-6, +inf == +inf
  elite set .................................... bitwise on the same J; end-to-end unless a
                                                 certified near-tie (oracle gap <= 2e-4 rel)
  mean, var, u0 ................................ <= 1e-4 max(|ref|_inf, 1 N)
"""
import math

import numpy as np
import pytest

from paper_2403_11383_b200 import workloads as W

pytestmark = pytest.mark.gpu

RTOL_J, ATOL_J = 1e-4, 1e-6


@pytest.fixture(scope="module")
def B():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2403_11383_b200 import binding, build
    build.build()
    binding.load_library()
    return binding


def _ctrl(B, cfg, inputs, state=None):
    c = B.Controller(cfg)
    st = state or W.initial_distribution(cfg)
    for r, inp in enumerate(inputs):
        c.set_reference(r, inp["xref"])
        c.set_distribution(r, st["mean"], st["var"], st["freq_idx"])
    c.iter = st["iter"]
    return c


def _tol_vec(ref):
    return 1e-4 * max(float(np.max(np.abs(ref))), 1.0)


def _check_costs(Jg, Jo):
    Jg = np.asarray(Jg, dtype=np.float64)
    inf_o = ~np.isfinite(Jo)
    assert np.array_equal(~np.isfinite(Jg), inf_o), "divergence pattern differs"
    fin = ~inf_o
    err = np.abs(Jg[fin] - Jo[fin])
    bound = RTOL_J * np.abs(Jo[fin]) + ATOL_J
    bad = np.nonzero(err > bound)[0]
    assert bad.size == 0, f"{bad.size} costs off; worst rel {np.max(err / np.maximum(np.abs(Jo[fin]), 1e-30)):.3e}"
    return float(np.max(err / np.maximum(np.abs(Jo[fin]), 1e-12))) if fin.any() else 0.0


def _check_outputs(og, ro, cfg, check_var=True):
    D = 12 * cfg["knots"]
    assert og["status"] == ro.status
    assert og["freq_idx"] == ro.freq_idx
    np.testing.assert_array_equal(og["contact0"], ro.contact0)
    assert np.max(np.abs(og["mean"] - ro.mean)) <= _tol_vec(ro.mean)
    assert np.max(np.abs(og["u0"] - ro.u0)) <= _tol_vec(ro.u0)
    if check_var:
        assert np.max(np.abs(og["var"] - ro.var)) <= _tol_vec(ro.var)
    assert og["n_diverged"] == ro.n_diverged
    if math.isfinite(ro.j_min):
        assert abs(og["j_min"] - ro.j_min) <= RTOL_J * abs(ro.j_min) + ATOL_J
    assert og["mean"].shape == (D,)


# ---------------------------------------------------------------------------
# a1: noise and samples
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("which", ["c1", "c3"])
def test_noise_bitwise(B, orc, which):
    cfg, inputs = W.config1() if which == "c1" else W.config3("cem", K=3000)
    st = W.initial_distribution(cfg)
    c = _ctrl(B, cfg, inputs, st)
    K = cfg["n_samples"]
    z, th, f = c.debug_samples(0, 0, K)
    r = orc.step(cfg, 0, inputs[0], dict(st))
    np.testing.assert_array_equal(z.view(np.uint32), r.z.view(np.uint32))
    np.testing.assert_array_equal(f, r.fidx)
    # theta2 = mu' + sigma z: the binary32 warm shift leaves an absolute error ~ ulp(mu')
    mu_s = orc.warm_shift(cfg, st["mean"])
    assert np.all(np.abs(th - r.theta) <= 1e-6 * (np.abs(r.theta) + np.abs(mu_s)[None, :] + 1.0))
    if which == "c3":
        assert set(np.unique(f)) == {0, 1, 2}


def test_noise_bitwise_nonzero_iter_and_robot(B, orc):
    cfg, inputs = W.config3("naive", K=700)
    cfg = dict(cfg, n_robots=3)
    inputs = [W.robot_input(cfg, r) for r in range(3)]
    st = W.initial_distribution(cfg)
    st["iter"] = 123456
    st["mean"] = st["mean"] + np.linspace(-5, 5, 48)
    c = _ctrl(B, cfg, inputs, st)
    for robot in range(3):
        z, th, f = c.debug_samples(robot, 5, 600)
        mu_s = orc.warm_shift(cfg, st["mean"])
        for i in (0, 1, 77, 599):
            th_o, z_o, f_o = orc.sample(cfg, mu_s, st["var"], 0, 123456, robot, 5 + i)
            np.testing.assert_array_equal(z[i].view(np.uint32), z_o.view(np.uint32))
            assert f[i] == f_o
            assert np.all(np.abs(th[i] - th_o) <= 1e-6 * (np.abs(th_o) + np.abs(mu_s) + 1.0))


# ---------------------------------------------------------------------------
# a2-a7: whole iterations
# ---------------------------------------------------------------------------
def _run_pair(B, orc, cfg, inputs, n_steps=1, check_var=True):
    st = W.initial_distribution(cfg)
    c = _ctrl(B, cfg, inputs, st)
    worst = 0.0
    for it in range(n_steps):
        ro = orc.step(cfg, 0, inputs[0], st)
        status, outs = c.step(inputs)
        assert status == ro.status
        Jg = c.debug_costs()[0]
        worst = max(worst, _check_costs(Jg, ro.J))
        _check_outputs(outs[0], ro, cfg, check_var)
        # re-sync the GPU distribution to the oracle's (oracle -> GPU only)
        c.set_distribution(0, st["mean"], st["var"], st["freq_idx"])
        assert c.iter == st["iter"]
    return c, worst


def test_config1_mppi_three_iterations(B, orc):
    cfg, inputs = W.config1()
    _run_pair(B, orc, cfg, inputs, n_steps=3)


def test_config2_mppi_paper_settings(B, orc):
    cfg, inputs = W.config2()
    _run_pair(B, orc, cfg, inputs, n_steps=2)


@pytest.mark.parametrize("mode", ["cem", "naive"])
def test_config3_three_iterations(B, orc, mode):
    cfg, inputs = W.config3(mode, K=3000)
    _run_pair(B, orc, cfg, inputs, n_steps=3)


@pytest.mark.parametrize("K", [1, 2, 127, 128, 129, 1000, 4097])
def test_ragged_sample_counts(B, orc, K):
    cfg, inputs = W.config2(K=K)
    _run_pair(B, orc, cfg, inputs)


@pytest.mark.parametrize("P,H", [(2, 12), (3, 7), (5, 12), (8, 20)])
def test_knot_and_horizon_variants(B, orc, P, H):
    cfg = W.base_config(n_samples=300, knots=P, horizon=H, gait_adapt=1)
    inputs = [W.robot_input(cfg, 0, cmd=(0.3, -0.2, 0.0), phase=W.q32(0.8))]
    _run_pair(B, orc, cfg, inputs)


@pytest.mark.parametrize("mode,scales", [("naive", [0.5, 1.0, 2.0]), ("mppi", [1.0, 0.25]), ("cem", [2.0, 1.0, 0.0])])
def test_multiple_gaussians(B, orc, mode, scales):
    """Naive's multiple Gaussian distributions (L41): sample k uses sigma_scale[k mod G]."""
    cfg = W.base_config(n_samples=900, mode=mode, n_elite=90 if mode == "cem" else 1, gait_adapt=1,
                        sigma_scale=scales)
    inputs = [W.robot_input(cfg, 0, cmd=(0.2, 0.1, 0.0), phase=W.q32(0.4))]
    st = W.initial_distribution(cfg)
    c = _ctrl(B, cfg, inputs, st)
    z, th, f = c.debug_samples(0, 0, 900)
    r = orc.step(cfg, 0, inputs[0], dict(st))
    np.testing.assert_array_equal(z.view(np.uint32), r.z.view(np.uint32))
    mu_s = orc.warm_shift(cfg, st["mean"])
    assert np.all(np.abs(th - r.theta) <= 1e-6 * (np.abs(r.theta) + np.abs(mu_s)[None, :] + 1.0))
    _run_pair(B, orc, cfg, inputs, n_steps=2)


@pytest.mark.parametrize("gait", ["pace", "bound", "fine_grid"])
def test_gait_variants(B, orc, gait):
    """f4: other periodic gaits and a finer theta1 grid are configuration ("a more
    fine-grained discretization step can be employed"; P:301 pacing)."""
    kw = dict(pace=dict(phase_offset=[0.0, 0.5, 0.0, 0.5]),
              bound=dict(phase_offset=[0.0, 0.0, 0.5, 0.5], duty_factor=0.4),
              fine_grid=dict(freq_hz=[1.3, 1.45, 1.6, 1.75, 1.9, 2.05, 2.2, 2.4]))[gait]
    cfg = W.base_config(n_samples=800, mode="naive", gait_adapt=1, **kw)
    inputs = [W.robot_input(cfg, 0, cmd=(0.3, 0.0, 0.0), phase=W.q32(0.15))]
    c, _ = _run_pair(B, orc, cfg, inputs, n_steps=2)
    if gait == "fine_grid":
        _, _, f = c.debug_samples(0, 0, 800)
        assert set(np.unique(f)) == set(range(8))


def test_maximum_horizon_and_knots(B, orc):
    """The largest supported shape: H = 64 steps (SBS_MAX_HORIZON), P = 8 knots (D = 96).
    Full stance and a small sigma keep the 1.28 s rollouts upright, away from the
    divergence thresholds (L35: near them the +inf decision is a binary32-vs-binary64
    discontinuity that a long open-loop horizon amplifies)."""
    cfg = W.base_config(n_samples=300, knots=8, horizon=64, gait_adapt=1, mode="naive", sigma=[1.0, 1.0, 2.0],
                        duty_factor=1.0)
    inputs = [W.robot_input(cfg, 0, cmd=(0.0, 0.0, 0.0), phase=W.q32(0.6))]
    _run_pair(B, orc, cfg, inputs)


def test_mppi_small_lambda_is_the_argmin_sample(B):
    """North star: MPPI as lambda -> 0 returns the argmin sample."""
    cfg, inputs = W.config2(K=3000)
    cfg = dict(cfg, **{"lambda": 1e-6})
    c = _ctrl(B, cfg, inputs)
    _, th, _ = c.debug_samples(0, 0, 3000)
    _, outs = c.step(inputs)
    J = c.debug_costs()[0]
    kmin = int(np.argmin(J))
    np.testing.assert_allclose(outs[0]["mean"], th[kmin], rtol=0, atol=1e-4 * max(np.max(np.abs(th[kmin])), 1.0))


def test_cem_all_samples_elite_is_the_population(B, orc):
    """K_e = K: CEM's update is the population mean and (floored) variance."""
    cfg, inputs = W.config3("cem", K=500)
    cfg = dict(cfg, n_elite=500)
    _run_pair(B, orc, cfg, inputs, n_steps=2)


def test_full_inertia_and_no_warm_shift(B, orc):
    cfg = W.base_config(n_samples=500, inertia=[0.135, 0.01, -0.02, 0.01, 0.54, 0.03, -0.02, 0.03, 0.58],
                        warm_shift=0, elite_preserve=0, duty_factor=1.0)
    inputs = [W.robot_input(cfg, 0, cmd=(0.2, 0.0, 0.0))]
    _run_pair(B, orc, cfg, inputs)


def _certified_near_tie(J, Ke):
    s = np.sort(np.where(np.isfinite(J), J, np.inf))
    if Ke >= len(s):
        return False
    a, b = s[Ke - 1], s[Ke]
    return np.isfinite(a) and abs(b - a) <= 2e-4 * abs(a)


@pytest.mark.parametrize("mode", ["cem", "naive"])
def test_config3_elites(B, orc, mode):
    cfg, inputs = W.config3(mode)
    st = W.initial_distribution(cfg)
    c = _ctrl(B, cfg, inputs, st)
    ro = orc.step(cfg, 0, inputs[0], st)
    status, outs = c.step(inputs)
    Jg = c.debug_costs()[0]
    _check_costs(Jg, ro.J)
    Ke = 1 if mode == "naive" else cfg["n_elite"]
    eg = c.debug_elites(0)
    if _certified_near_tie(ro.J, Ke):
        pytest.skip("certified near-tie at the elite boundary")
    np.testing.assert_array_equal(np.sort(eg), np.sort(ro.elite))
    _check_outputs(outs[0], ro, cfg, check_var=True)


def test_select_same_J_bitwise(B, orc):
    rng = np.random.default_rng(21)
    # (16384, 12000): the compacted list exceeds the shared-memory staging (direct writes)
    for K, Ke in [(1, 1), (64, 1), (64, 64), (1000, 100), (10000, 1000), (16384, 10000), (16384, 12000),
                  (12000, 11999), (50000, 3), (70001, 7000)]:
        for kind in ("ties", "uniform", "signed"):
            if kind == "ties":
                J = rng.integers(0, 25, K).astype(np.float32)
            elif kind == "signed":
                J = rng.normal(0.0, 5.0, K).astype(np.float32)
            else:
                J = rng.uniform(0, 10, K).astype(np.float32)
            J[rng.integers(0, K, max(1, K // 50))] = np.inf
            J[rng.integers(0, K, max(1, K // 100))] = np.nan
            if K > 2:
                J[0] = -0.0
                J[1] = 0.0
            e_g = B.debug_select(J, Ke)
            e_o = orc.cem_select(J.astype(np.float64), Ke)
            np.testing.assert_array_equal(e_g, np.sort(e_o))


def test_all_diverged_and_singular(B, orc):
    cfg, inputs = W.config1()
    st = W.initial_distribution(cfg)
    c = _ctrl(B, cfg, inputs, st)
    bad = dict(inputs[0])
    x0 = bad["x0"].copy()
    x0[3] = 1e8
    bad["x0"] = x0
    status, outs = c.step([bad])
    assert status == 1 and outs[0]["n_diverged"] == cfg["n_samples"]
    m, v, f = c.get_distribution(0)
    np.testing.assert_array_equal(m, np.float32(st["mean"]))
    x0 = inputs[0]["x0"].copy()
    x0[7] = 1.5699
    with pytest.raises(B.SBSError) as e:
        c.step([dict(inputs[0], x0=x0)])
    assert e.value.status == -2
    x0[7] = np.nan
    with pytest.raises(B.SBSError) as e:
        c.step([dict(inputs[0], x0=x0)])
    assert e.value.status == -3


def test_batched_robots_match_oracle(B, orc):
    R = 5
    cfg = W.base_config(n_samples=300, n_robots=R, gait_adapt=1)
    rng = np.random.default_rng(3)
    inputs = [W.robot_input(cfg, r, cmd=(rng.uniform(-.5, .5), rng.uniform(-.5, .5), 0), phase=int(rng.integers(0, 2**32)))
              for r in range(R)]
    c = B.Controller(cfg)
    st0 = W.initial_distribution(cfg)
    for r in range(R):
        c.set_reference(r, inputs[r]["xref"])
    status, outs = c.step(inputs)
    Jg = c.debug_costs()
    for r in range(R):
        st = dict(st0)
        ro = orc.step(cfg, r, inputs[r], st)
        _check_costs(Jg[r], ro.J)
        _check_outputs(outs[r], ro, cfg)


@pytest.mark.parametrize("mode", ["cem", "naive", "mppi"])
def test_batched_robots_two_steps_all_modes(B, orc, mode):
    """R = 3 robots through the host path (captured graph, iteration counter in device
    memory): two consecutive iterations against the oracle, per robot."""
    R = 3
    cfg = W.base_config(n_samples=600, n_robots=R, gait_adapt=1, mode=mode, n_elite=60 if mode == "cem" else 1)
    rng = np.random.default_rng(11)
    inputs = [W.robot_input(cfg, r, cmd=(rng.uniform(-.5, .5), rng.uniform(-.5, .5), 0), phase=int(rng.integers(0, 2**32)))
              for r in range(R)]
    c = B.Controller(cfg)
    states = [W.initial_distribution(cfg) for _ in range(R)]
    for r in range(R):
        c.set_reference(r, inputs[r]["xref"])
    for it in range(2):
        status, outs = c.step(inputs)
        Jg = c.debug_costs()
        for r in range(R):
            ro = orc.step(cfg, r, inputs[r], states[r])
            _check_costs(Jg[r], ro.J)
            if mode != "mppi" and _certified_near_tie(ro.J, 1 if mode == "naive" else cfg["n_elite"]):
                continue
            _check_outputs(outs[r], ro, cfg)
            c.set_distribution(r, states[r]["mean"], states[r]["var"], states[r]["freq_idx"])  # oracle -> GPU
        assert c.iter == it + 1


def test_host_path_equals_device_path(B):
    """sbs_step (one robot: inputs and reference inside the kernel parameters) and
    sbs_step_device (inputs in device memory) run the same arithmetic: bitwise equal."""
    import ctypes as C

    import torch
    for cfg, inputs in (W.config2(K=3000), W.config3("cem", K=3000), W.config3("naive", K=3000)):
        a = _ctrl(B, cfg, inputs)
        b = _ctrl(B, cfg, inputs)
        d_in = torch.from_numpy(np.frombuffer(bytes(B.make_inputs(inputs)), dtype=np.uint8).copy()).cuda()
        d_out = torch.zeros(C.sizeof(B.sbs_output), dtype=torch.uint8, device="cuda")
        for _ in range(2):
            _, oa = a.step(inputs)
            b.step_device(d_in.data_ptr(), d_out.data_ptr(), torch.cuda.current_stream().cuda_stream)
            torch.cuda.synchronize()
            ob = B.output_dict(B.sbs_output.from_buffer_copy(d_out.cpu().numpy().tobytes()), 48)
            for key in ("mean", "var", "u0"):
                np.testing.assert_array_equal(oa[0][key], ob[key])
            assert oa[0]["iter"] == ob["iter"] and oa[0]["freq_idx"] == ob["freq_idx"]


@pytest.mark.parametrize("mode", ["mppi", "naive", "cem"])
@pytest.mark.parametrize("H", [12, 7, 24, 40])
def test_latency_mode_variants_are_bitwise_equal(B, mode, H, monkeypatch):
    """The latency-mode rollout with and without the producer / integrator warp split
    (SBS_AB: 12 warps tabulate the stance-leg forces while 4 warps run RK4) computes the
    same bits: costs, means, elites.  The throughput-mode rollout (one thread per sample,
    its own instruction schedule and MPPI reduction order) agrees to rounding."""
    base = W.config3(mode, K=3000) if mode != "mppi" else W.config2(K=3000)
    cfg, inputs = base
    cfg = dict(cfg, horizon=H)
    inputs = [W.robot_input(cfg, 0, cmd=(0.4, 0.0, 0.1))]
    res = {}
    for tag, env in (("ab", {}), ("split", {"SBS_AB": "0"}), ("plain", {"SBS_SPLIT": "0"})):
        for k in ("SBS_AB", "SBS_SPLIT"):
            monkeypatch.delenv(k, raising=False)
        for k, v in env.items():
            monkeypatch.setenv(k, v)
        c = _ctrl(B, cfg, inputs)
        outs = [c.step(inputs)[1][0] for _ in range(2)]
        res[tag] = (c.debug_costs().copy(), outs, c.debug_elites(0).copy() if mode == "cem" else None)
    np.testing.assert_array_equal(res["split"][0], res["ab"][0])
    for oa, ob in zip(res["split"][1], res["ab"][1]):
        for key in ("mean", "var", "u0"):
            np.testing.assert_array_equal(oa[key], ob[key])
    if mode == "cem":
        np.testing.assert_array_equal(res["split"][2], res["ab"][2])
    if H > 12:  # long horizons amplify rounding differences chaotically (divergence threshold)
        return
    Ja, Jp = res["ab"][0], res["plain"][0]
    assert np.array_equal(np.isfinite(Ja), np.isfinite(Jp))
    f = np.isfinite(Ja)
    assert np.all(np.abs(Ja[f] - Jp[f]) <= 1e-4 * np.abs(Jp[f]) + 1e-6)
    o_a, o_p = res["ab"][1][0], res["plain"][1][0]           # first iteration: same distribution in
    for key in ("mean", "u0"):
        assert np.max(np.abs(o_a[key] - o_p[key])) <= 1e-4 * max(float(np.max(np.abs(o_p[key]))), 1.0)


def test_host_path_completion_flag(B, monkeypatch):
    """sbs_step (one robot) waits on the mapped flag its finishing CTA raises; the same
    steps waited with cudaStreamSynchronize (SBS_POLL=0) give the same outputs, for
    every mode, and device_us is measured only with profiling on."""
    for cfg, inputs in (W.config2(K=3000), W.config3("cem", K=3000), W.config3("naive", K=3000)):
        res = []
        for poll in ("1", "0"):
            monkeypatch.setenv("SBS_POLL", poll)
            c = _ctrl(B, cfg, inputs)
            outs = [c.step(inputs)[1][0] for _ in range(3)]
            assert all(o["device_us"] == 0.0 for o in outs)
            res.append(outs)
        for oa, ob in zip(*res):
            for key in ("mean", "var", "u0"):
                np.testing.assert_array_equal(oa[key], ob[key])
            assert oa["iter"] == ob["iter"]
        c.profile(True)
        assert c.step(inputs)[1][0]["device_us"] > 0.0


def test_reference_from_device_memory(B):
    """sbs_set_reference_device (device buffer, stream-ordered) is the same reference as
    sbs_set_reference for both the host path and the device path."""
    import torch
    cfg, inputs = W.config2(K=2000)
    xr = np.asarray(inputs[0]["xref"], dtype=np.float32)
    a = _ctrl(B, cfg, inputs)
    b = _ctrl(B, cfg, inputs)
    b.set_reference(0, np.zeros_like(xr))                     # overwritten below
    d_x = torch.from_numpy(xr.copy()).cuda()
    b.set_reference_device(d_x.data_ptr(), torch.cuda.current_stream().cuda_stream)
    np.testing.assert_array_equal(b.get_reference(0), xr)
    _, oa = a.step(inputs)
    _, ob = b.step(inputs)
    np.testing.assert_array_equal(oa[0]["mean"], ob[0]["mean"])
    np.testing.assert_array_equal(a.debug_costs(), b.debug_costs())


def test_determinism_and_checkpoint(B):
    cfg, inputs = W.config2(K=5000)
    a = _ctrl(B, cfg, inputs)
    b = _ctrl(B, cfg, inputs)
    _, oa = a.step(inputs)
    _, ob = b.step(inputs)
    for key in ("mean", "u0", "var"):
        np.testing.assert_array_equal(oa[0][key], ob[0][key])
    np.testing.assert_array_equal(a.debug_costs(), b.debug_costs())
    snap = a.get_state()
    _, o1 = a.step(inputs)
    a.set_state(snap)
    _, o2 = a.step(inputs)
    np.testing.assert_array_equal(o1[0]["mean"], o2[0]["mean"])


# ---------------------------------------------------------------------------
# full BASELINE sizes, in the launch configuration bench.py times
# ---------------------------------------------------------------------------
def test_config4_full_size_sampled(B, orc):
    K = 1 << 22
    cfg, inputs = W.config4(K)
    st = W.initial_distribution(cfg)
    c = _ctrl(B, cfg, inputs, st)
    status, outs = c.step(inputs)
    Jg = c.debug_costs()[0]
    rng = np.random.default_rng(4)
    ks = np.concatenate([[0, 1, K - 1], rng.integers(0, K, 150)])
    mu_s = orc.warm_shift(cfg, st["mean"])
    inp = inputs[0]
    Jo = np.array([orc.rollout(cfg, inp["x0"], inp["phase"], inp["feet_cur"], inp["feet_next"], inp["xref"],
                               orc.sample(cfg, mu_s, st["var"], 0, 0, 0, int(k))[0], 0) for k in ks])
    _check_costs(Jg[ks], Jo)
    # properties at full size: beta = min J; mean inside the samples' hull; ESS in [1, K]
    assert outs[0]["j_min"] == np.min(Jg)
    assert 1.0 <= outs[0]["ess"] <= K
    assert np.all(np.isfinite(outs[0]["mean"]))


def test_config5_full_size_sampled(B, orc):
    cfg, inputs = W.config5()
    c = B.Controller(cfg)
    for r in range(cfg["n_robots"]):
        c.set_reference(r, inputs[r]["xref"])
    status, outs = c.step(inputs)
    Jg = c.debug_costs()
    st0 = W.initial_distribution(cfg)
    mu_s = orc.warm_shift(cfg, st0["mean"])
    rng = np.random.default_rng(5)
    for r in rng.integers(0, cfg["n_robots"], 12):
        inp = inputs[int(r)]
        ks = rng.integers(0, cfg["n_samples"], 8)
        Jo = np.array([orc.rollout(cfg, inp["x0"], inp["phase"], inp["feet_cur"], inp["feet_next"], inp["xref"],
                                   orc.sample(cfg, mu_s, st0["var"], 0, 0, int(r), int(k))[0], 0) for k in ks])
        _check_costs(Jg[int(r)][ks], Jo)
    # two whole robots against the oracle iteration
    for r in (0, cfg["n_robots"] - 1):
        ro = orc.step(cfg, r, inputs[r], dict(st0))
        _check_costs(Jg[r], ro.J)
        _check_outputs(outs[r], ro, cfg)


@pytest.mark.parametrize("K,world", [(10000, 2), (4097, 2), (8192, 4), (1 << 19, 2), (3 << 18, 2)])  # (2^19: dynamic tiles per rank, tree-aligned slices; 3 * 2^18: not aligned)
def test_sharded_mppi_records_match_single_gpu(B, orc, K, world):
    """The world > 1 kernels (rank record + rank-order merge) on one GPU: `world`
    contexts each roll out their slice and emit a record, the records are
    concatenated in rank order (what the NCCL all-gather does) and every rank
    finishes the iteration; all ranks agree with each other and with world = 1."""
    import ctypes as C

    import torch
    cfg, inputs = W.config2(K=K)
    st = W.initial_distribution(cfg)
    arr = B.make_inputs(inputs)
    d_in = torch.from_numpy(np.frombuffer(bytes(arr), dtype=np.uint8).copy()).cuda()
    ranks = [B.Controller(cfg, rank=g, world=world) for g in range(world)]
    for c in ranks:
        c.set_reference(0, inputs[0]["xref"])
    nrec = ranks[0].record_floats()
    recs = torch.zeros((world, nrec), dtype=torch.float32, device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    slices = [c.local_range() for c in ranks]
    assert slices[0][0] == 0 and sum(kl for _, kl in slices) == K
    for g, c in enumerate(ranks):
        c.step_records(d_in.data_ptr(), recs[g].data_ptr(), s)
    outs = []
    for c in ranks:
        d_out = torch.zeros(C.sizeof(B.sbs_output), dtype=torch.uint8, device="cuda")
        c.finish_records(recs.data_ptr(), d_in.data_ptr(), d_out.data_ptr(), s)
        torch.cuda.synchronize()
        o = B.sbs_output.from_buffer_copy(d_out.cpu().numpy().tobytes())
        outs.append(B.output_dict(o, 48))
    for o in outs[1:]:
        np.testing.assert_array_equal(o["mean"], outs[0]["mean"])
        assert o["freq_idx"] == outs[0]["freq_idx"]
    J = np.concatenate([c.debug_costs()[0] for c in ranks])
    single = _ctrl(B, cfg, inputs, st)
    _, so = single.step(inputs)
    np.testing.assert_array_equal(J, single.debug_costs()[0])       # same samples, same costs
    assert outs[0]["j_min"] == so[0]["j_min"] and outs[0]["n_diverged"] == so[0]["n_diverged"]
    assert np.max(np.abs(outs[0]["mean"] - so[0]["mean"])) <= 1e-5 * max(np.max(np.abs(so[0]["mean"])), 1.0)
    ro = orc.step(cfg, 0, inputs[0], dict(st))
    _check_outputs(outs[0], ro, cfg)
    assert all(c.iter == 1 for c in ranks)


@pytest.mark.parametrize("mode,K,world,ke", [("cem", 10000, 2, 1000), ("cem", 10000, 4, 2500), ("cem", 4099, 3, 37),
                                             ("cem", 40000, 2, 3000), ("naive", 10000, 2, 1), ("naive", 5003, 4, 1)])
def test_sharded_cem_naive_records_match_single_gpu(B, orc, mode, K, world, ke):
    """Sample-sharded CEM / Naive on one GPU through the caller-driven
    exchange: every rank offers its K_e smallest (J, k) (CEM) or its argmin
    (Naive); after the rank-order merge every rank holds the same elite set and
    distribution, bitwise equal to world = 1 (same costs, same exact selection,
    same regenerated elites and moment order), and within tolerance of the oracle."""
    import ctypes as C

    import torch
    cfg, inputs = W.config3(mode, K=K)
    cfg = dict(cfg, n_elite=ke)
    st = W.initial_distribution(cfg)
    arr = B.make_inputs(inputs)
    d_in = torch.from_numpy(np.frombuffer(bytes(arr), dtype=np.uint8).copy()).cuda()
    ranks = [B.Controller(cfg, rank=g, world=world) for g in range(world)]
    for c in ranks:
        c.set_reference(0, inputs[0]["xref"])
    nrec = ranks[0].record_floats()
    assert nrec % 4 == 0 and nrec >= 8 + (2 * ke if mode == "cem" else 0)
    recs = torch.zeros((world, nrec), dtype=torch.float32, device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    for g, c in enumerate(ranks):
        c.step_records(d_in.data_ptr(), recs[g].data_ptr(), s)
    outs, elites = [], []
    for c in ranks:
        d_out = torch.zeros(C.sizeof(B.sbs_output), dtype=torch.uint8, device="cuda")
        c.finish_records(recs.data_ptr(), d_in.data_ptr(), d_out.data_ptr(), s)
        torch.cuda.synchronize()
        o = B.sbs_output.from_buffer_copy(d_out.cpu().numpy().tobytes())
        outs.append(B.output_dict(o, 48))
        elites.append(c.debug_elites(0))
    single = _ctrl(B, cfg, inputs, st)
    _, so = single.step(inputs)
    J = np.concatenate([c.debug_costs()[0] for c in ranks])
    np.testing.assert_array_equal(J, single.debug_costs()[0])
    e1 = single.debug_elites(0)
    for o, e in zip(outs, elites):
        np.testing.assert_array_equal(e, e1)                       # same global elite set, index order
        np.testing.assert_array_equal(o["mean"], so[0]["mean"])    # bitwise: same elites, same order
        np.testing.assert_array_equal(o["var"], so[0]["var"])
        np.testing.assert_array_equal(o["u0"], so[0]["u0"])
        assert o["freq_idx"] == so[0]["freq_idx"] and o["j_min"] == so[0]["j_min"]
        assert o["n_diverged"] == so[0]["n_diverged"]
        assert abs(o["j_mean"] - so[0]["j_mean"]) <= 1e-5 * abs(so[0]["j_mean"])  # rank-grouped sum
    # the elite set is the exact K_e smallest (J, k) of the concatenated costs
    order = np.lexsort((np.arange(K), np.where(np.isfinite(J), J, np.inf)))
    np.testing.assert_array_equal(np.sort(order[:ke]), e1)
    ro = orc.step(cfg, 0, inputs[0], dict(st))
    _check_outputs(outs[0], ro, cfg)
    assert all(c.iter == 1 for c in ranks)


def test_sharded_cem_rejects_too_few_samples_per_rank(B):
    cfg, _ = W.config3("cem", K=1000)
    with pytest.raises(Exception):
        B.Controller(dict(cfg, n_elite=600), rank=0, world=2)


@pytest.mark.parametrize("mode,K,world,ke,R", [("mppi", 10000, 2, 1, 1), ("mppi", 65536, 4, 1, 1), ("naive", 6000, 2, 1, 1),
                                               ("cem", 12000, 3, 800, 1), ("mppi", 4000, 2, 1, 3), ("cem", 4000, 2, 300, 2)])
def test_peer_memory_exchange_matches_single_gpu(B, orc, mode, K, world, ke, R):
    """The rank-record exchange over peer memory (finishing CTA stores into every peer's
    buffer + flag; streams wait on the flags in the front end; no NCCL), here with `world`
    contexts of one process on one GPU, each on its own stream and enqueued in rank order
    (the waits are stream-front-end waits, no kernel waits on another).  Three consecutive
    iterations (both exchange buffers); every rank agrees bitwise with the others, and with
    world = 1 (CEM / Naive bitwise, MPPI within 1e-5: its cross-rank sums regroup)."""
    import ctypes as C

    import torch
    if mode == "mppi":
        cfg, _ = W.config2(K=K)
    else:
        cfg, _ = W.config3(mode, K=K)
        cfg = dict(cfg, n_elite=ke)
    cfg = dict(cfg, n_robots=R)
    inputs = [W.robot_input(cfg, r, cmd=(0.4, 0.1 * r, 0.0), phase=W.q32(0.3 + 0.2 * r)) for r in range(R)]
    d_in = torch.from_numpy(np.frombuffer(bytes(B.make_inputs(inputs)), dtype=np.uint8).copy()).cuda()
    ranks = [B.Controller(cfg, rank=g, world=world) for g in range(world)]
    bases = [c.peer_handle()[1] for c in ranks]
    for c in ranks:
        for r in range(R):
            c.set_reference(r, inputs[r]["xref"])
        c.peer_connect(bases=bases)
    streams = [torch.cuda.Stream() for _ in ranks]
    n_out = C.sizeof(B.sbs_output)
    outs = [torch.zeros(R * n_out, dtype=torch.uint8, device="cuda") for _ in ranks]
    single = B.Controller(cfg)
    for r in range(R):
        single.set_reference(r, inputs[r]["xref"])
    torch.cuda.synchronize()
    for it in range(3):
        for g, c in enumerate(ranks):
            c.step_device(d_in.data_ptr(), outs[g].data_ptr(), streams[g].cuda_stream)
        torch.cuda.synchronize()
        _, so = single.step(inputs)
        for r in range(R):
            res = [B.output_dict(B.sbs_output.from_buffer_copy(o.cpu().numpy().tobytes()[r * n_out:(r + 1) * n_out]), 48)
                   for o in outs]
            for o in res[1:]:
                np.testing.assert_array_equal(o["mean"], res[0]["mean"])
                np.testing.assert_array_equal(o["var"], res[0]["var"])
                assert o["freq_idx"] == res[0]["freq_idx"]
            if mode == "mppi":
                assert np.max(np.abs(res[0]["mean"] - so[r]["mean"])) <= 1e-5 * max(np.max(np.abs(so[r]["mean"])), 1.0)
                # keep the single-GPU context on the ranks' distribution (the regrouped sums differ in the last bits)
                m, v, f = ranks[0].get_distribution(r)
                single.set_distribution(r, m, v, f)
            else:
                np.testing.assert_array_equal(res[0]["mean"], so[r]["mean"])
                np.testing.assert_array_equal(res[0]["var"], so[r]["var"])
                np.testing.assert_array_equal(ranks[0].debug_elites(r), single.debug_elites(r))
            assert res[0]["j_min"] == so[r]["j_min"] and res[0]["n_diverged"] == so[r]["n_diverged"]
    assert all(c.iter == 3 for c in ranks)


def test_peer_disconnect_falls_back_to_the_caller_exchange(B):
    """After sbs_peer_connect(NULL, NULL) the contexts are back on the caller-driven exchange."""
    import ctypes as C

    import torch
    cfg, inputs = W.config2(K=4000)
    d_in = torch.from_numpy(np.frombuffer(bytes(B.make_inputs(inputs)), dtype=np.uint8).copy()).cuda()
    ranks = [B.Controller(cfg, rank=g, world=2) for g in range(2)]
    bases = [c.peer_handle()[1] for c in ranks]
    for c in ranks:
        c.set_reference(0, inputs[0]["xref"])
        c.peer_connect(bases=bases)
    outs = [torch.zeros(C.sizeof(B.sbs_output), dtype=torch.uint8, device="cuda") for _ in ranks]
    streams = [torch.cuda.Stream() for _ in ranks]
    for g, c in enumerate(ranks):
        c.step_device(d_in.data_ptr(), outs[g].data_ptr(), streams[g].cuda_stream)
    torch.cuda.synchronize()
    for c in ranks:
        c.peer_connect()
    with pytest.raises(Exception):                       # no NCCL, no peers: the host step refuses
        ranks[0].step_device(d_in.data_ptr(), outs[0].data_ptr(), 0)
    recs = torch.zeros((2, ranks[0].record_floats()), dtype=torch.float32, device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    for g, c in enumerate(ranks):
        c.step_records(d_in.data_ptr(), recs[g].data_ptr(), s)
    for g, c in enumerate(ranks):
        c.finish_records(recs.data_ptr(), d_in.data_ptr(), outs[g].data_ptr(), s)
    torch.cuda.synchronize()
    a, b = (B.output_dict(B.sbs_output.from_buffer_copy(o.cpu().numpy().tobytes()), 48) for o in outs)
    np.testing.assert_array_equal(a["mean"], b["mean"])
    assert all(c.iter == 2 for c in ranks)
