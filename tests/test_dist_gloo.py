"""Multi-process (world_size 2, gloo, CPU) coverage of the sample-sharded path.

What runs on N GPUs: every rank samples and rolls out its slice of the global
sample indices (the counter RNG makes the noise independent of the sharding),
reduces it to one MPPI record (beta_r, sum w, sum w^2, sum w theta relative to
beta_r) and the ranks' records are all-gathered and merged in rank order.  Here
the per-rank work is done by the CPU oracle and the exchange by gloo; the merged
result must equal the single-process oracle iteration.  CEM / Naive: every rank
offers its K_e smallest (J, k) (Naive: K_e = 1), the offers are all-gathered in
rank order (= global index order) and the K_e smallest of the world * K_e
candidates are the global elite set.  Also covered: the NCCL unique-id
bootstrap through torch.distributed.
"""
import math
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2403_11383_b200 import workloads as W
from paper_2403_11383_b200.dist import bootstrap_nccl_id, shard_range


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _record(J, theta, lam):
    """Rank record of the MPPI exchange (exact restatement of the kernel's merge algebra)."""
    beta = np.min(J) if len(J) else math.inf
    if not math.isfinite(beta):
        return np.concatenate([[math.inf, 0.0, 0.0], np.zeros(theta.shape[1])])
    w = np.exp(-(J - beta) / lam)
    return np.concatenate([[beta, w.sum(), (w * w).sum()], w @ theta])


def _merge(records, lam):
    beta = min(r[0] for r in records)
    S = V = 0.0
    for r in records:                       # fixed rank order
        sc = math.exp(-(r[0] - beta) / lam) if math.isfinite(r[0]) else 0.0
        S = S + r[1] * sc
        V = V + r[3:] * sc
    return V / S, beta


def _worker(rank, world, port, cfg, inp, out_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import Oracle
    orc = Oracle()
    K, D = cfg["n_samples"], 12 * cfg["knots"]
    st = W.initial_distribution(cfg)
    mu_s = orc.warm_shift(cfg, st["mean"])
    k0, kl = shard_range(K, rank, world)
    J = np.zeros(kl)
    th = np.zeros((kl, D))
    for i in range(kl):
        th[i], _, f = orc.sample(cfg, mu_s, st["var"], 0, 0, 0, k0 + i)
        J[i] = orc.rollout(cfg, inp["x0"], inp["phase"], inp["feet_cur"], inp["feet_next"], inp["xref"], th[i], f)
    rec = torch.tensor(_record(J, th, cfg["lambda"]), dtype=torch.float64)
    recs = [torch.zeros_like(rec) for _ in range(world)]
    dist.all_gather(recs, rec)
    mean, beta = _merge([r.numpy() for r in recs], cfg["lambda"])
    nid = bootstrap_nccl_id(rank)
    out_q.put((rank, mean, beta, k0, kl, nid))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("K", [257, 1000])
def test_two_rank_mppi_equals_single_process(orc, K):
    cfg, inputs = W.config2(K=K)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, cfg, inputs[0], q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=300) for _ in procs], key=lambda t: t[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    st = W.initial_distribution(cfg)
    ro = orc.step(cfg, 0, inputs[0], st)
    # shards tile [0, K) in rank order
    assert res[0][3] == 0 and res[0][3] + res[0][4] == res[1][3] and res[1][3] + res[1][4] == K
    for rank, mean, beta, _, _, nid in res:
        np.testing.assert_allclose(mean, ro.mean, rtol=0, atol=1e-10 * max(1, np.max(np.abs(ro.mean))))
        assert beta == ro.j_min
    assert res[0][5] == res[1][5] and len(res[0][5]) == 128      # same ncclUniqueId on both ranks


def test_shard_range_matches_library_formula():
    for K in (1, 2, 7, 10000, 2 ** 22 + 3):
        for world in (1, 2, 3, 4, 8):
            if K < world:
                continue
            slices = [shard_range(K, r, world) for r in range(world)]
            assert slices[0][0] == 0
            assert all(slices[i][0] + slices[i][1] == slices[i + 1][0] for i in range(world - 1))
            assert slices[-1][0] + slices[-1][1] == K
            assert max(s[1] for s in slices) - min(s[1] for s in slices) <= 1


def _cem_worker(rank, world, port, cfg, inp, out_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import Oracle
    orc = Oracle()
    K, D = cfg["n_samples"], 12 * cfg["knots"]
    ke = 1 if cfg["mode"] == "naive" else cfg["n_elite"]
    st = W.initial_distribution(cfg)
    mu_s = orc.warm_shift(cfg, st["mean"])
    k0, kl = shard_range(K, rank, world)
    J = np.zeros(kl)
    for i in range(kl):
        th, _, f = orc.sample(cfg, mu_s, st["var"], 0, 0, 0, k0 + i)
        J[i] = orc.rollout(cfg, inp["x0"], inp["phase"], inp["feet_cur"], inp["feet_next"], inp["xref"], th, f)
    loc = np.sort(orc.cem_select(J, ke))                          # local K_e smallest, index order
    offer = torch.tensor(np.concatenate([J[loc], (k0 + loc).astype(np.float64)]), dtype=torch.float64)
    offers = [torch.zeros_like(offer) for _ in range(world)]
    dist.all_gather(offers, offer)
    cand_J = np.concatenate([o.numpy()[:ke] for o in offers])     # rank order = global index order
    cand_k = np.concatenate([o.numpy()[ke:] for o in offers]).astype(np.int64)
    assert np.all(np.diff(cand_k) > 0)
    elite = cand_k[orc.cem_select(cand_J, ke)]                    # (J, position) order = (J, k) order
    out_q.put((rank, elite))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("mode,K,ke", [("cem", 400, 50), ("cem", 301, 150), ("naive", 300, 1)])
def test_two_rank_cem_elites_equal_single_process(orc, mode, K, ke):
    cfg, inputs = W.config3(mode, K=K)
    cfg = dict(cfg, n_elite=ke)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_cem_worker, args=(r, 2, port, cfg, inputs[0], q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=300) for _ in procs], key=lambda t: t[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    ro = orc.step(cfg, 0, inputs[0], W.initial_distribution(cfg))
    for _, elite in res:
        np.testing.assert_array_equal(elite, ro.elite[:ke])       # same set, same rank order
