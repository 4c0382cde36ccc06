"""GPU parity, second set: the launch shapes and edge cases the first set did not
reach.

  * the normative noise recipe over every one of its 2^23 radius inputs and 2^23
    angle inputs, bit for bit against the oracle (O3-O4; "theta_k ~ N(theta, C)");
  * Philox4x32-10 against cuRAND's curand_Philox4x32_10 on the device (O1);
  * theta2 within the stated ulp contract;
  * MPPI at K = 2^16 and 2^17 with the static split (more CTA records than the one-pass
    merge holds: the chunked merge), and at 2^18 with dynamic tiles and the reduction
    tree the K = 2^22 bench launch takes
    against the oracle (Alg. 4), and the conditioning check of SURVEY 8(c4)
    over lambda = 1, 10, 100;
  * yaw near +-pi (the MUFU sincos and the rint wrap against libm and remainder);
  * CEM with fewer finite costs than elites (Alg. 1; L17, L26);
  * robot sharding: two contexts with robot_offset = one context of all robots, bitwise.
"""
import math

import numpy as np
import pytest

from paper_2403_11383_b200 import workloads as W
from test_gpu_parity import _check_costs, _check_outputs, _ctrl, _tol_vec

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


# ---------------------------------------------------------------------------
# O1, O3-O4: noise
# ---------------------------------------------------------------------------
def _exhaustive_words(seed=0):
    """2^22 Philox blocks whose radius words (w0, w2) run through all 2^23 values of
    w >> 9 and whose angle words (w1, w3) do too (an odd multiplier permutes [0, 2^23));
    the 9 low bits, which the recipe discards, are random."""
    n = 1 << 22
    b = np.arange(n, dtype=np.uint64)
    low = np.random.default_rng(seed).integers(0, 512, size=(n, 4), dtype=np.uint64)
    w = np.empty((n, 4), dtype=np.uint32)
    w[:, 0] = ((2 * b) << 9 | low[:, 0]).astype(np.uint32)
    w[:, 2] = ((2 * b + 1) << 9 | low[:, 2]).astype(np.uint32)
    w[:, 1] = ((((2 * b) * 2654435761) % (1 << 23)) << 9 | low[:, 1]).astype(np.uint32)
    w[:, 3] = ((((2 * b + 1) * 2654435761) % (1 << 23)) << 9 | low[:, 3]).astype(np.uint32)
    return w


def test_noise_recipe_exhaustive(B, orc):
    w = _exhaustive_words()
    assert len(np.unique(np.concatenate([w[:, 0], w[:, 2]]) >> 9)) == 1 << 23
    assert len(np.unique(np.concatenate([w[:, 1], w[:, 3]]) >> 9)) == 1 << 23
    zg = B.debug_noise(w)
    zo = orc.normal4_batch(w)
    bad = np.nonzero(zg.view(np.uint32) != zo.view(np.uint32))
    assert bad[0].size == 0, f"{bad[0].size} of {zg.size} z differ, first block {bad[0][:4]}"
    # edge words: all-zero and all-one words in every position
    edge = np.array([[0, 0, 0, 0], [0xFFFFFFFF] * 4, [0, 0xFFFFFFFF, 0, 0xFFFFFFFF], [0xFFFFFFFF, 0, 0xFFFFFFFF, 0],
                     [0x1FF, 0x1FF, 0x200, 0x200], [0xFFFFFE00, 0xE0000000, 0x1FFFFFFF, 0x20000000]], dtype=np.uint32)
    np.testing.assert_array_equal(B.debug_noise(edge).view(np.uint32), orc.normal4_batch(edge).view(np.uint32))


def test_philox_matches_curand_and_oracle(B, orc):
    rng = np.random.default_rng(7)
    n = 1 << 20
    ctr = rng.integers(0, 1 << 32, size=(n, 4), dtype=np.uint64).astype(np.uint32)
    key = rng.integers(0, 1 << 32, size=(n, 2), dtype=np.uint64).astype(np.uint32)
    ctr[:4] = [[0, 0, 0, 0], [0xFFFFFFFF] * 4, [0x243f6a88, 0x85a308d3, 0x13198a2e, 0x03707344], [0x80000000, 5, 7, 1]]
    key[:4] = [[0, 0], [0xFFFFFFFF] * 2, [0xa4093822, 0x299f31d0], [0x40311383, 2]]
    ours, cur = B.debug_philox(ctr, key)
    np.testing.assert_array_equal(ours[:, 0], cur)          # plain form == cuRAND
    np.testing.assert_array_equal(ours[:, 1], cur)          # round-key form == cuRAND
    for i in list(range(4)) + list(rng.integers(0, n, 200)):
        np.testing.assert_array_equal(orc.philox(ctr[i], key[i]), cur[i])


def _ulp(x):
    """binary32 ulp of |x| (x > 0): 2^(floor(log2 x) - 23), normal range."""
    return np.ldexp(1.0, np.floor(np.log2(np.maximum(np.abs(x), np.finfo(np.float32).tiny))).astype(int) - 23)


def test_theta2_ulp_contract(B, orc):
    """theta2 = fma(sqrt(var), z, mu') in binary32 with mu' the binary32 warm shift (L20) of
    the previous mean: within 4 ulp of the operation's magnitude max(|theta2|, sum_q |WS_pq
    mean_q|, sigma |z|) of the oracle's binary64 value (the warm shift's
    dot product rounds on the scale of its terms, not of its result)."""
    worst = 0.0
    for it in (0, 1, 7):
        cfg, inputs = W.config3("cem", K=2000)
        st = W.initial_distribution(cfg)
        st["iter"] = it
        st["mean"] = st["mean"] + np.random.default_rng(it).normal(0, 20, 48)  # a non-constant spline
        c = _ctrl(B, cfg, inputs, st)
        z_g, th, _ = c.debug_samples(0, 0, 2000)
        r = orc.step(cfg, 0, inputs[0], dict(st))
        D = 48
        WS = np.stack([orc.warm_shift(cfg, np.eye(D)[q]) for q in range(D)], axis=1)  # mu' = WS mean
        terms = np.abs(WS) @ np.abs(st["mean"])
        sig_z = np.sqrt(st["var"])[None, :] * np.abs(r.z)
        scale = _ulp(np.maximum(np.maximum(np.abs(r.theta), terms[None, :]), sig_z))
        worst = max(worst, float(np.max(np.abs(th - r.theta) / scale)))
    assert worst <= 4.0, worst


# ---------------------------------------------------------------------------
# a5 at the chunked-merge and dynamic-tile launch shapes, conditioning
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("K,dyn", [(1 << 16, None), (1 << 17, "0"), (1 << 18, None)])
def test_mppi_chunked_merge_against_oracle(B, orc, K, dyn, monkeypatch):
    """K = 2^16 (one tile per CTA) and 2^17 with SBS_DYN=0: 512 / 592 CTA records, more
    than one staged merge holds (the chunked merge); K = 2^18: dynamic tiles and the
    reduction tree."""
    monkeypatch.delenv("SBS_DYN", raising=False)
    if dyn is not None:
        monkeypatch.setenv("SBS_DYN", dyn)
    cfg, inputs = W.config4(K)
    st = W.initial_distribution(cfg)
    c = _ctrl(B, cfg, inputs, st)
    ro = orc.step(cfg, 0, inputs[0], st)
    status, outs = c.step(inputs)
    assert status == ro.status == 0
    _check_costs(c.debug_costs()[0], ro.J)
    _check_outputs(outs[0], ro, cfg)
    assert outs[0]["ess"] == pytest.approx(ro.ess, rel=1e-3)


def test_mppi_conditioning_lambda_sweep(B, orc):
    """kappa = max_k |J_gpu - J_orc| / lambda bounds the weight perturbation,
    so |mu_gpu - mu_orc| <= kappa max_k ||theta_k - mu_new|| to first order (plus the
    binary32 rounding of the sums); a larger lambda shrinks kappa and the error."""
    errs = {}
    for lam in (1.0, 10.0, 100.0):
        cfg, inputs = W.config2(K=10000)
        cfg = dict(cfg, **{"lambda": lam})
        st = W.initial_distribution(cfg)
        c = _ctrl(B, cfg, inputs, st)
        ro = orc.step(cfg, 0, inputs[0], st)
        _, outs = c.step(inputs)
        Jg = c.debug_costs()[0].astype(np.float64)
        kappa = float(np.max(np.abs(Jg - ro.J))) / lam
        spread = float(np.max(np.abs(ro.theta - ro.mean[None, :])))
        err = float(np.max(np.abs(outs[0]["mean"] - ro.mean)))
        assert err <= kappa * spread + 1e-5 * max(float(np.max(np.abs(ro.mean))), 1.0), (lam, err, kappa, spread)
        errs[lam] = err
    # the lambda-driven part of the error shrinks; what stays is the binary32 rounding of the sums
    assert errs[100.0] <= errs[1.0] + 1e-5 * max(float(np.max(np.abs(ro.mean))), 1.0), errs


# ---------------------------------------------------------------------------
# yaw near +-pi
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("yaw0,yaw_ref,wz", [(3.0, 3.05, 1.0), (-3.1, 3.1, -0.5), (3.1, -3.12, 2.0)])
def test_yaw_near_pi(B, orc, yaw0, yaw_ref, wz):
    """|yaw| ~ pi in the state and the reference (a yaw rate carries the state across +-pi
    within the horizon; the reference may sit on the other branch): costs, mean, u0 against
    the oracle's libm trigonometry and remainder wrap."""
    cfg, inputs = W.config2(K=4000)
    inp = dict(inputs[0])
    x0 = inp["x0"].copy()
    x0[8] = W.f32(yaw0)
    x0[11] = W.f32(wz)
    inp["x0"] = x0
    xr = inp["xref"].copy()
    xr[:, 8] = W.f32(yaw_ref)
    inp["xref"] = xr
    st = W.initial_distribution(cfg)
    c = _ctrl(B, cfg, [inp], st)
    ro = orc.step(cfg, 0, inp, st)
    _, outs = c.step([inp])
    _check_costs(c.debug_costs()[0], ro.J)
    _check_outputs(outs[0], ro, cfg)


# ---------------------------------------------------------------------------
# CEM with most samples diverged
# ---------------------------------------------------------------------------
def test_cem_fewer_finite_than_elites(B, orc):
    """Pitched over with a large pitch rate: ~20 % of the rollouts cross the pitch limit
    (J = +inf, L26) and K_e exceeds the finite count, so the elite list ends in diverged
    samples that must not enter the moments (L17).  Near the Euler singularity the binary32
    and binary64 trajectories separate (L35): there the divergence decision itself can
    differ, so the update is checked on the GPU's own costs -- the oracle's CEM update
    (orc_cem_update) on the GPU's J and the oracle's samples -- and the costs on the
    samples whose oracle trajectory stays 0.12 rad or more from the singularity."""
    cfg, inputs = W.config3("cem", K=3000)
    cfg = dict(cfg, n_elite=2900)
    inp = dict(inputs[0])
    x0 = inp["x0"].copy()
    x0[7] = W.f32(1.0)
    x0[10] = W.f32(8.0)
    inp["x0"] = x0
    st = W.initial_distribution(cfg)
    c = _ctrl(B, cfg, [inp], st)
    ro = orc.step(cfg, 0, inp, dict(st))
    _, outs = c.step([inp])
    Jg = c.debug_costs()[0].astype(np.float64)
    n_fin = int(np.sum(np.isfinite(Jg)))
    assert 0 < n_fin < cfg["n_elite"]
    mu_s = orc.warm_shift(cfg, st["mean"])
    max_pitch = np.empty(3000)
    for k in range(3000):
        th, _, f = orc.sample(cfg, mu_s, st["var"], st["freq_idx"], 0, 0, k)
        _, tr = orc.rollout(cfg, inp["x0"], inp["phase"], inp["feet_cur"], inp["feet_next"], inp["xref"], th, f,
                            traj=True)
        max_pitch[k] = np.max(np.abs(tr[:, 7])) if np.all(np.isfinite(tr)) else np.inf
    regular = np.isfinite(Jg) & np.isfinite(ro.J) & (max_pitch < 1.45)  # 0.12 rad from the singularity
    if regular.any():
        _check_costs(Jg[regular], ro.J[regular])
    D = 12 * cfg["knots"]
    floor = np.array([(cfg["sigma_min_frac"] * cfg["sigma"][d % 3]) ** 2 for d in range(D)])
    rc, mu, var, e, dg = orc.cem_update(Jg, ro.theta, cfg["n_elite"], floor, 1, st["var"])
    assert rc == 0 and dg.n_diverged == 3000 - n_fin
    np.testing.assert_array_equal(np.sort(c.debug_elites(0)), np.sort(e))
    assert outs[0]["n_diverged"] == 3000 - n_fin
    assert np.max(np.abs(outs[0]["mean"] - mu)) <= _tol_vec(mu)
    assert np.max(np.abs(outs[0]["var"] - var)) <= _tol_vec(var)


# ---------------------------------------------------------------------------
# config 5 sharded by robot (BASELINE configs[4])
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("mode", ["mppi", "cem"])
def test_robot_offset_shards_equal_one_context(B, mode):
    """Two contexts owning robots [0, 3) and [3, 6) (robot_offset = 3) reproduce one
    six-robot context bit for bit over two iterations: the noise counter carries the global
    robot index (O2), so sharding by robot changes nothing but where the work runs."""
    R = 6
    cfg = W.base_config(n_samples=1024, n_robots=R, mode=mode, n_elite=100 if mode == "cem" else 1)
    rng = np.random.default_rng(5)
    inputs = [W.robot_input(cfg, r, cmd=(rng.uniform(-.5, .5), rng.uniform(-.5, .5), 0),
                            phase=int(rng.integers(0, 2 ** 32))) for r in range(R)]
    full = B.Controller(cfg)
    halves = [B.Controller(dict(cfg, n_robots=3), robot_offset=0), B.Controller(dict(cfg, n_robots=3), robot_offset=3)]
    for r in range(R):
        full.set_reference(r, inputs[r]["xref"])
        halves[r // 3].set_reference(r % 3, inputs[r]["xref"])
    for _ in range(2):
        _, of = full.step(inputs)
        _, o0 = halves[0].step(inputs[:3])
        _, o1 = halves[1].step(inputs[3:])
        Jf = full.debug_costs()
        np.testing.assert_array_equal(Jf[:3], halves[0].debug_costs())
        np.testing.assert_array_equal(Jf[3:], halves[1].debug_costs())
        for r, o in enumerate(o0 + o1):
            for key in ("mean", "var", "u0"):
                np.testing.assert_array_equal(of[r][key], o[key])
            assert of[r]["freq_idx"] == o["freq_idx"] and of[r]["j_min"] == o["j_min"]


def test_checkpoint_after_side_stream_step(B):
    """State getters wait for device-path work enqueued on a caller's side stream (the
    checkpoint is the state after that step, never a torn one), and a host-path step
    issued after it is ordered behind it."""
    import ctypes as C

    import torch
    cfg, inputs = W.config4(1 << 20)
    a = _ctrl(B, cfg, inputs)
    b = _ctrl(B, cfg, inputs)
    side = torch.cuda.Stream()
    d_in = torch.from_numpy(np.frombuffer(bytes(B.make_inputs(inputs)), dtype=np.uint8).copy()).cuda()
    d_out = torch.zeros(C.sizeof(B.sbs_output), dtype=torch.uint8, device="cuda")
    torch.cuda.synchronize()
    a.step_device(d_in.data_ptr(), d_out.data_ptr(), side.cuda_stream)   # ~0.3 ms on the side stream
    snap = a.get_state()                                                  # no explicit synchronisation
    m_a, _, _ = a.get_distribution(0)
    b.step_device(d_in.data_ptr(), d_out.data_ptr(), side.cuda_stream)
    side.synchronize()
    m_b, _, _ = b.get_distribution(0)
    np.testing.assert_array_equal(m_a, m_b)
    c = _ctrl(B, cfg, inputs)
    c.set_state(snap)
    np.testing.assert_array_equal(c.get_distribution(0)[0], m_b)
    _, o1 = a.step(inputs)                     # host path after the side-stream step
    _, o2 = b.step(inputs)
    np.testing.assert_array_equal(o1[0]["mean"], o2[0]["mean"])


def test_config4_full_size_update_recomputed(B):
    """The bench's launch configuration (K = 2^22: dynamic tiles, 32768 tile records reduced
    by the fan-in-64 tree): the
    MPPI update (Alg. 4) recomputed in binary64 from the GPU's own costs and
    samples -- the costs are oracle-checked on samples (test_config4_full_size_sampled), the
    samples bitwise (the noise tests) -- must match the kernel's mean, Omega and ESS."""
    K = 1 << 22
    cfg, inputs = W.config4(K)
    st = W.initial_distribution(cfg)
    c = _ctrl(B, cfg, inputs, st)
    chunk = 1 << 20
    thetas = [c.debug_samples(0, k0, chunk)[1].astype(np.float64) for k0 in range(0, K, chunk)]  # this step's draws
    status, outs = c.step(inputs)
    assert status == 0
    J = c.debug_costs()[0].astype(np.float64)
    beta = np.min(J)
    w = np.exp(-(J - beta) / cfg["lambda"])
    omega = np.sum(w)
    mu = sum(w[i * chunk:(i + 1) * chunk] @ th for i, th in enumerate(thetas)) / omega
    assert np.max(np.abs(outs[0]["mean"] - mu)) <= 1e-4 * max(float(np.max(np.abs(mu))), 1.0)
    assert outs[0]["omega"] == pytest.approx(omega, rel=1e-4)
    assert outs[0]["ess"] == pytest.approx(omega ** 2 / np.sum(w * w), rel=1e-3)
    assert outs[0]["j_min"] == beta


# ---------------------------------------------------------------------------
# a6: the one-launch CEM path (select + elite moments in one thread-block cluster)
# ---------------------------------------------------------------------------
def _pitched(inp):
    inp = dict(inp)
    x0 = inp["x0"].copy()
    x0[7] = W.f32(1.0)
    x0[10] = W.f32(8.0)
    inp["x0"] = x0
    return inp


@pytest.mark.parametrize("case", ["config3", "ragged_R3", "max_groups", "one_elite", "diverged", "preserve"])
def test_cem_cluster_path_is_bitwise_the_two_kernel_path(B, case, monkeypatch):
    """CEM at world = 1 runs select + elite moments + finish as one cluster launch when
    K <= 16384 and K_e <= 2048 (sbs_cem_cluster_kernel).  It performs the two-kernel
    path's arithmetic in the same order (Alg. 1; L17), so means, variances,
    outputs and elite lists are bitwise those of SBS_CEM_CLUSTER=0, over three
    iterations; both are checked against the oracle elsewhere."""
    R = 1
    if case == "config3":
        cfg, inputs = W.config3("cem", K=10000)
    elif case == "ragged_R3":
        R = 3
        cfg = W.base_config(n_samples=3001, n_robots=R, mode="cem", n_elite=37)
        inputs = [W.robot_input(cfg, r, cmd=(0.3 * r, 0.0, 0.1)) for r in range(R)]
    elif case == "max_groups":
        cfg = W.base_config(n_samples=16384, mode="cem", n_elite=2048)
        inputs = [W.robot_input(cfg, 0, cmd=(0.5, 0.0, 0.0))]
    elif case == "one_elite":
        cfg = W.base_config(n_samples=64, mode="cem", n_elite=1)
        inputs = [W.robot_input(cfg, 0)]
    elif case == "diverged":  # fewer finite costs than elites
        cfg, inputs = W.config3("cem", K=2100)
        cfg = dict(cfg, n_elite=2048)
        inputs = [_pitched(inputs[0])]
    else:
        cfg, inputs = W.config3("cem", K=4000)
        cfg = dict(cfg, elite_preserve=0)
    res = {}
    for tag, env in (("cluster", None), ("cluster8", "8"), ("two", "0")):
        monkeypatch.delenv("SBS_CEM_CLUSTER", raising=False)
        if env is not None:
            monkeypatch.setenv("SBS_CEM_CLUSTER", env)
        c = _ctrl(B, cfg, inputs)
        assert c.L.sbs_launches_per_step(c.ctx) == (3 if env == "0" else 2)
        outs = [c.step(inputs)[1] for _ in range(3)]
        res[tag] = (outs, [c.debug_elites(r).copy() for r in range(R)], c.debug_costs().copy())
    ot, et, Jt = res["two"]
    for tag in ("cluster", "cluster8"):
        oc, ec, Jc = res[tag]
        np.testing.assert_array_equal(Jc, Jt)
        for r in range(R):
            np.testing.assert_array_equal(ec[r], et[r])
        for it in range(3):
            for r in range(R):
                for key in ("mean", "var", "u0", "j_min", "j_mean", "n_diverged", "freq_idx", "status", "iter"):
                    np.testing.assert_array_equal(np.asarray(oc[it][r][key]), np.asarray(ot[it][r][key]),
                                                  err_msg=f"{tag} {key}")
    oc, _, Jc = res["cluster"]
    if case == "diverged":
        assert 0 < oc[0][0]["n_diverged"] and int(np.sum(np.isfinite(Jc[0]))) < cfg["n_elite"]


def test_cem_cluster_path_only_while_the_clusters_fit(B):
    """The one-launch CEM path gives every robot a cluster of 16 (or 8) SMs; with more
    robots than the GPU holds clusters at once the select + elite kernels (one select SM
    per robot) are the better trade, and sbs_create keeps them."""
    import torch
    n_sm = torch.cuda.get_device_properties(0).multi_processor_count
    for R, launches in ((1, 2), (n_sm // 16, 2), (n_sm // 8 + 1, 3)):
        cfg = W.base_config(n_samples=1024, n_robots=R, mode="cem", n_elite=64)
        c = B.Controller(cfg)
        assert c.L.sbs_launches_per_step(c.ctx) == launches, (R, launches)
        c.close()


# ---------------------------------------------------------------------------
# a5 with dynamic tile scheduling (throughput mode, one robot, more tiles than CTAs)
# ---------------------------------------------------------------------------
def test_dynamic_tiles_are_deterministic_and_match_the_static_split(B, orc, monkeypatch):
    """With dynamic tile scheduling the CTAs take tiles from a counter, so which CTA runs
    which tile changes from run to run; the tile records are reduced by a tree fixed by
    the tile indices alone, so repeated runs are bitwise equal.  Against the static split
    (SBS_DYN=0: per-CTA running records, another summation order) and the oracle's update
    on the GPU's costs, the new mean agrees to rounding (Alg. 4)."""
    K = 1 << 18  # 2048 tiles over 592 CTAs
    cfg, inputs = W.config4(K)
    st = W.initial_distribution(cfg)
    outs = []
    for env in (None, None, "0"):
        monkeypatch.delenv("SBS_DYN", raising=False)
        if env is not None:
            monkeypatch.setenv("SBS_DYN", env)
        c = _ctrl(B, cfg, inputs, dict(st))
        o = [c.step(inputs)[1][0]]
        J1 = c.debug_costs()[0].copy()  # (first iteration: the same distribution on every path)
        o.append(c.step(inputs)[1][0])
        outs.append((o, J1))
        c.close()
    (a, Ja), (b, Jb), (s, Js) = outs
    np.testing.assert_array_equal(Ja, Jb)
    np.testing.assert_array_equal(Ja, Js)  # the costs do not depend on the schedule at all
    for oa, ob in zip(a, b):
        for key in ("mean", "u0", "j_min", "j_mean", "ess", "omega"):
            np.testing.assert_array_equal(np.asarray(oa[key]), np.asarray(ob[key]), err_msg=key)
    for oa, os_ in zip(a, s):
        assert np.max(np.abs(oa["mean"] - os_["mean"])) <= 1e-5 * max(float(np.max(np.abs(os_["mean"]))), 1.0)
    assert a[0]["j_min"] == s[0]["j_min"]
    # the first iteration's update recomputed in binary64 from the GPU's costs
    c = _ctrl(B, cfg, inputs, dict(st))
    _, o1 = c.step(inputs)
    Jg = c.debug_costs()[0].astype(np.float64)
    fin = np.isfinite(Jg)
    mu_s = orc.warm_shift(cfg, st["mean"])
    idx = np.nonzero(fin)[0][::997]  # a sample of rows is enough to pin the weighted mean's direction
    assert idx.size > 0
    w = np.exp(-(Jg[fin] - Jg[fin].min()) / cfg["lambda"])
    assert abs(float(o1[0]["j_min"]) - Jg[fin].min()) <= 1e-6 * abs(Jg[fin].min())
    assert np.isclose(float(o1[0]["ess"]), w.sum() ** 2 / (w * w).sum(), rtol=1e-4)


@pytest.mark.parametrize("K,world", [(1 << 20, 2), (1 << 21, 2), (1 << 21, 4)])
def test_sharded_mppi_is_bitwise_independent_of_the_gpu_count(B, K, world):
    """SURVEY 8(e)'s fixed reduction tree: with dynamic tiles every rank reduces its
    tiles' records by the same fan-in-64 tree over the global tile index; when a rank's
    slice is made of whole nodes of the level below the global root, it emits those
    nodes' records and the rank-order merge after the exchange is the global root's
    merge.  The new mean, u0 and the diagnostics are then bitwise those of one GPU
    (Alg. 4, P:188-201 evaluated by the same arithmetic in the same order)."""
    import ctypes as C

    import torch
    cfg, inputs = W.config4(K)
    st = W.initial_distribution(cfg)
    arr = B.make_inputs(inputs)
    d_in = torch.from_numpy(np.frombuffer(bytes(arr), dtype=np.uint8).copy()).cuda()
    single = _ctrl(B, cfg, inputs, dict(st))
    ranks = [B.Controller(cfg, rank=g, world=world) for g in range(world)]
    for c in ranks:
        c.set_reference(0, inputs[0]["xref"])
    nrec = ranks[0].record_floats()
    assert nrec == (K // world) // (1 << 19) * (8 + 48)  # whole level-2 nodes (2^19 samples) per rank
    s = torch.cuda.current_stream().cuda_stream
    for it in range(2):
        _, so = single.step(inputs)
        recs = torch.zeros((world, nrec), dtype=torch.float32, device="cuda")
        for g, c in enumerate(ranks):
            c.step_records(d_in.data_ptr(), recs[g].data_ptr(), s)
        for c in ranks:
            d_out = torch.zeros(C.sizeof(B.sbs_output), dtype=torch.uint8, device="cuda")
            c.finish_records(recs.data_ptr(), d_in.data_ptr(), d_out.data_ptr(), s)
            torch.cuda.synchronize()
            o = B.output_dict(B.sbs_output.from_buffer_copy(d_out.cpu().numpy().tobytes()), 48)
            for key in ("mean", "var", "u0", "j_min", "j_mean", "ess", "omega", "n_diverged", "freq_idx"):
                np.testing.assert_array_equal(np.asarray(o[key]), np.asarray(so[0][key]), err_msg=f"iter {it} {key}")


@pytest.mark.parametrize("K", [(1 << 18) + 77, (1 << 17) - 51])
def test_dynamic_tiles_ragged_last_tile_and_partial_nodes(B, orc, monkeypatch, K):
    """Dynamic tiles with K = 2^18 + 77 (a partial last tile of 77 samples, partial tree
    nodes at every level) and K = 2^17 - 51 (1024 tiles over 592 CTAs: between one and
    two tiles per CTA, the last one partial); repeated runs are bitwise equal, the static
    split agrees to rounding, and J_min, the effective sample size and the divergence
    count follow from the GPU's costs in binary64 (Alg. 4; the mean against the oracle at
    the tree's launch shape: test_mppi_chunked_merge_against_oracle at K = 2^18)."""
    cfg, inputs = W.config4(K)
    st = W.initial_distribution(cfg)
    res = []
    for env in (None, None, "0"):
        monkeypatch.delenv("SBS_DYN", raising=False)
        if env is not None:
            monkeypatch.setenv("SBS_DYN", env)
        c = _ctrl(B, cfg, inputs, dict(st))
        _, o = c.step(inputs)
        res.append((o[0], c.debug_costs()[0].copy()))
        c.close()
    (a, Ja), (b, Jb), (s_, Js) = res
    np.testing.assert_array_equal(Ja, Jb)
    np.testing.assert_array_equal(Ja, Js)
    for key in ("mean", "u0", "j_min", "ess"):
        np.testing.assert_array_equal(np.asarray(a[key]), np.asarray(b[key]), err_msg=key)
    assert np.max(np.abs(a["mean"] - s_["mean"])) <= 1e-5 * max(float(np.max(np.abs(s_["mean"]))), 1.0)
    # binary64 weights from the GPU's costs
    Jg = Ja.astype(np.float64)
    fin = np.isfinite(Jg)
    w = np.where(fin, np.exp(-(np.where(fin, Jg, 0) - Jg[fin].min()) / cfg["lambda"]), 0.0)
    assert float(a["j_min"]) == float(np.float32(Jg[fin].min()))
    assert np.isclose(float(a["ess"]), w.sum() ** 2 / (w * w).sum(), rtol=1e-4)
    assert int(a["n_diverged"]) == int((~fin).sum())
