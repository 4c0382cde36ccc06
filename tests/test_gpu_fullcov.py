"""GPU parity of full-covariance CEM (DESIGN reading L42) against
the oracle: noise bitwise, theta2 = mu' + L z within binary32 accumulation error,
costs / elites / mean / var / the new Cholesky factor within the DESIGN sec. 5
tolerances, sharding invariance, checkpoint round trip."""
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


def _cfg(K=1500, Ke=150, P=4):
    cfg, inputs = W.config3("cem", K=K)
    cfg = dict(cfg, n_elite=Ke, full_cov=1, knots=P)
    inputs = [W.robot_input(cfg, 0, cmd=(0.0, 0.1, 0.0), push=(0.5, 0.08))]
    return cfg, inputs


def _near_tie(J, Ke):
    s = np.sort(np.where(np.isfinite(J), J, np.inf))
    return Ke < len(s) and np.isfinite(s[Ke - 1]) and abs(s[Ke] - s[Ke - 1]) <= 2e-4 * abs(s[Ke - 1])


def _sync(c, st, D):
    c.set_distribution(0, st["mean"], st["var"], st["freq_idx"])
    Lm = np.asarray(st["chol"])
    c.set_covariance(0, Lm @ Lm.T)
    c.iter = st["iter"]


@pytest.mark.parametrize("P", [4, 2])
def test_full_covariance_iterations_match_oracle(B, orc, P):
    cfg, inputs = _cfg(P=P)
    D = 12 * P
    st = W.initial_distribution(cfg)
    c = B.Controller(cfg)
    c.set_reference(0, inputs[0]["xref"])
    _sync(c, st, D)
    checked = 0
    for it in range(4):
        Lo = np.asarray(st["chol"]).copy()
        z, th, _ = c.debug_samples(0, 0, 400)
        ro = orc.step(cfg, 0, inputs[0], st)
        np.testing.assert_array_equal(z.view(np.uint32), ro.z[:400].view(np.uint32))
        scale = np.abs(ro.theta[:400]) + np.abs(Lo).sum(1)[None, :] * 4.0 + 1.0
        assert np.all(np.abs(th - ro.theta[:400]) <= 1e-5 * scale), it
        status, outs = c.step(inputs)
        assert status == ro.status
        Jg = c.debug_costs()[0]
        fin = np.isfinite(ro.J)
        assert np.array_equal(np.isfinite(Jg), fin)
        assert np.all(np.abs(Jg[fin] - ro.J[fin]) <= 1e-4 * np.abs(ro.J[fin]) + 1e-6)
        if _near_tie(ro.J, cfg["n_elite"]):                # certified near-tie: elites may differ
            _sync(c, st, D)
            continue
        checked += 1
        np.testing.assert_array_equal(c.debug_elites(0), np.sort(ro.elite))
        o = outs[0]
        tol = lambda ref: 1e-4 * max(float(np.max(np.abs(ref))), 1.0)   # noqa: E731
        assert np.max(np.abs(o["mean"] - ro.mean)) <= tol(ro.mean)
        assert np.max(np.abs(o["var"] - ro.var)) <= tol(ro.var)
        assert np.max(np.abs(o["u0"] - ro.u0)) <= tol(ro.u0)
        Lg = c.get_cholesky(0)
        Lo_new = np.asarray(st["chol"])
        assert np.max(np.abs(Lg - Lo_new)) <= tol(Lo_new), it
        assert np.all(np.triu(Lg, 1) == 0)
        _sync(c, st, D)                                    # oracle -> GPU only
    assert checked >= 2


def test_full_covariance_sharded_is_world_invariant(B):
    import torch
    cfg, inputs = _cfg(K=8000, Ke=800)
    arr = B.make_inputs(inputs)
    d_in = torch.from_numpy(np.frombuffer(bytes(arr), dtype=np.uint8).copy()).cuda()
    single = B.Controller(cfg)
    single.set_reference(0, inputs[0]["xref"])
    _, so = single.step(inputs)
    ranks = [B.Controller(cfg, rank=g, world=2) for g in range(2)]
    for c in ranks:
        c.set_reference(0, inputs[0]["xref"])
    nrec = ranks[0].record_floats()
    recs = torch.zeros((2, nrec), dtype=torch.float32, device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    for g, c in enumerate(ranks):
        c.step_records(d_in.data_ptr(), recs[g].data_ptr(), s)
    for c in ranks:
        d_out = torch.zeros(C.sizeof(B.sbs_output), dtype=torch.uint8, device="cuda")
        c.finish_records(recs.data_ptr(), d_in.data_ptr(), d_out.data_ptr(), s)
        torch.cuda.synchronize()
        o = B.output_dict(B.sbs_output.from_buffer_copy(d_out.cpu().numpy().tobytes()), 48)
        np.testing.assert_array_equal(o["mean"], so[0]["mean"])
        np.testing.assert_array_equal(o["var"], so[0]["var"])
        np.testing.assert_array_equal(c.get_cholesky(0), single.get_cholesky(0))


def test_full_covariance_checkpoint_roundtrip(B):
    cfg, inputs = _cfg(K=2000, Ke=200)
    a = B.Controller(cfg)
    a.set_reference(0, inputs[0]["xref"])
    a.step(inputs)
    blob = a.get_state()
    b = B.Controller(cfg)
    b.set_reference(0, inputs[0]["xref"])
    b.set_state(blob)
    np.testing.assert_array_equal(a.get_cholesky(0), b.get_cholesky(0))
    _, oa = a.step(inputs)
    _, ob = b.step(inputs)
    np.testing.assert_array_equal(oa[0]["mean"], ob[0]["mean"])
    np.testing.assert_array_equal(a.get_cholesky(0), b.get_cholesky(0))


def test_set_covariance_rejects_indefinite(B):
    cfg, _ = _cfg(K=500, Ke=50)
    c = B.Controller(cfg)
    with pytest.raises(Exception):
        c.set_covariance(0, -np.eye(48))
    with pytest.raises(Exception):
        B.Controller(dict(cfg, mode="mppi"))                   # full_cov is a CEM option
