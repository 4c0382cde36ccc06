#!/usr/bin/env python
"""Benchmark of one SBS MPC iteration (arxiv 2403.11383) on B200.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl sbs|reference]
                  [--exchange peer|nccl] [--scaling strong|weak]

Headline workload: BASELINE.json configs[3], the large-batch MPPI iteration, at
K = 2^22 samples, H = 12, dt = 0.02 s, fixed trot (the largest single-GPU config;
SURVEY 8(d1)).  With N > 1 (torchrun, one process per GPU) the same K = 2^22
samples are sharded over the N ranks (strong scaling; `--scaling weak` keeps
2^22 samples per GPU instead); the ranks' (min, sum w, sum w theta) records are
exchanged over peer memory (each rank's finishing CTA stores its record into
every peer's buffer over NVLink; the peers' streams wait on a flag), or with one
NCCL all-gather (`--exchange nccl`).

One JSON line on rank 0.  `value` = sample-steps/s (K_total H / device time per
iteration, inputs resident in HBM, L2 flushed between timed iterations, max over
ranks); `e2e` = the same metric through the public host API (sbs_set_reference +
sbs_step with host buffers, host clock); `latency` = config 2 (BASELINE.json
configs[1], K = 10,000, the paper's settings) per-iteration device time and e2e;
`roofline` = the fused rollout kernel against the FP32 ALU peak, with the
algorithmic FLOPs per sample-step from the oracle's op-counting mode.
`--impl reference` times the CPU oracle (the reference arm of this tier) on a
bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

K_HEADLINE = 1 << 22          # BASELINE configs[3] at its largest single-GPU size
K_LATENCY = 10000             # BASELINE configs[1]
H = 12
# Algorithmic FLOPs per sample-step, frozen from the oracle's
# op-counting mode over the config-2 workload (scripts/op_count.py, 256 samples;
# tests/test_oracle_opcount.py re-derives them): the rollout + cost (a2-a4) alone,
# and the whole fused kernel (+ sampling a1: binary32 Box-Muller and theta2, + MPPI a5).
ALG_FLOP_ROLLOUT = 9343.0 / 12.0          # 778.58
ALG_FLOP_FUSED = 886.1419270833334        # rollout 778.58 + sampling 95.16 + MPPI 12.40
ALG_FLOP_PER_SAMPLE_STEP = ALG_FLOP_FUSED
FLOP_BREAKDOWN = {"rollout_a2_a4": ALG_FLOP_ROLLOUT, "sampling_a1": 95.15755208333333, "mppi_a5": 12.401041666666666,
                  "total": ALG_FLOP_FUSED, "unit": "FLOP per sample-step",
                  "source": "oracle op-counting mode (oracle/opcount.cpp, scripts/op_count.py), config 2 trot average"}
# per-kernel CUDA events (for the roofline's kernel time) bracket every PROFILE_EVERY-th
# timed step, so their own cost stays out of the headline per-iteration time
PROFILE_EVERY = 10
FP32_LANES_PER_SM = 128
METRIC = "sample-steps/sec and MPC-iteration latency (us) at N samples"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="sbs", choices=["sbs", "reference"])
    ap.add_argument("--exchange", default="peer", choices=["peer", "nccl"])
    ap.add_argument("--scaling", default="strong", choices=["strong", "weak"])
    ap.add_argument("--e2e-steps", type=int, default=100)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-other-configs", action="store_true", help="skip the config 2/3/5 lines (ncu launch lists)")
    ap.add_argument("--same-gpu", action="store_true",
                    help="code-path check only: every rank on device 0 (peer exchange between processes of one "
                         "GPU); its timings are not multi-GPU numbers")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", str(rank)))
    return rank, world, local


def k_total(args, world):
    return K_HEADLINE * (world if args.scaling == "weak" else 1)


def headline_config(args, world, exchange=None):
    """The `config` dict of the JSON line (shared by both arms, so they compare equal)."""
    K = k_total(args, world)
    par = "samples sharded over %d GPU(s)" % world
    if world > 1:
        par += ", rank records by " + (exchange or ("NCCL all-gather" if args.exchange == "nccl" else
                                                   "peer-memory stores (NVLink) + stream flag waits"))
    return {"workload": "config4: MPPI, K=%d samples, H=12, dt=0.02 s, fixed trot 1.3 Hz, cmd 0.5 m/s "
                        "(BASELINE.json configs[3], largest single-GPU size)" % K,
            "K_total": K, "K_per_gpu": K // world, "H": H, "mode": "mppi", "scaling": args.scaling,
            "parallelism": par, "l2": "flushed between timed iterations (256 MiB memset, outside the events)"}


# ---------------------------------------------------------------------------
# clocks during the timed region (B200_PROFILING.md recipe)
# ---------------------------------------------------------------------------
class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.path = None

    def start(self):
        fd, self.path = tempfile.mkstemp(prefix="sbs_clocks_", suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except OSError:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        rows = []
        for line in open(self.path):
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 9 and parts[1].isdigit():
                rows.append(parts)
        os.unlink(self.path)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        sm = [int(r[1]) for r in rows]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i].lower().startswith("active")})
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": int(rows[0][2]), "reasons": reasons,
                "samples": len(rows), "power_w_max": max(float(r[3]) for r in rows if r[3] not in ("", "[N/A]"))}


# ---------------------------------------------------------------------------
# CPU oracle timing (cpu_baseline leg and the reference arm)
# ---------------------------------------------------------------------------
def oracle_rate(K_sample: int, n_steps: int, warmup: int = 1, workload: str = "config4"):
    """Time the oracle as it stands (single thread): n_steps iterations of the workload's
    scenario on K_sample of its samples each.  Returns (sample-steps/s, per-step seconds)."""
    from oracle import Oracle
    from paper_2403_11383_b200 import workloads as W
    orc = Oracle()
    cfg, inputs = (W.config4 if workload == "config4" else W.config2)(K_sample)
    st = W.initial_distribution(cfg)
    for _ in range(warmup):
        orc.step(cfg, 0, inputs[0], st, keep=False)
    times = []
    for _ in range(n_steps):
        t = time.perf_counter()
        orc.step(cfg, 0, inputs[0], st, keep=False)
        times.append(time.perf_counter() - t)
    return K_sample * H * n_steps / sum(times), times


def _oracle_worker(args):
    K_sample, n_steps = args
    _, times = oracle_rate(K_sample, n_steps, warmup=0)
    return K_sample * H * n_steps, sum(times)


def oracle_rate_all_cores(K_sample: int, n_steps: int):
    """The same oracle iteration run concurrently in one process per host core (the oracle
    as it stands, parallelised by the harness only).  Returns (sample-steps/s over the wall
    time, processes)."""
    import multiprocessing as mp
    n = os.cpu_count() or 1
    ctx = mp.get_context("fork")
    t = time.perf_counter()
    with ctx.Pool(n) as pool:
        res = pool.map(_oracle_worker, [(K_sample, n_steps)] * n)
    wall = time.perf_counter() - t
    return sum(r[0] for r in res) / wall, n


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    # each step: a bounded sample of the config-4 iteration sized so the whole run takes ~1-3 minutes
    budget_s = 120.0
    per_sample_step_s = 0.6e-6
    n = max(args.steps + args.warmup, 1)
    K_s = int(max(64, min(65536, budget_s / (n * H * per_sample_step_s))))
    value, times = oracle_rate(K_s, args.steps, warmup=args.warmup)
    ms = 1e3 * sum(times) / len(times)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "sample-steps/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": args.scaling, "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": headline_config(args, world),
        "cpu_baseline": {"value": value, "unit": "sample-steps/s", "cores": 1, "kind": "oracle",
                         "sample": f"{K_s} of the {k_total(args, world)} samples of the config-4 iteration per "
                                   f"step (same scenario and seeds), {args.steps} steps, single thread"},
        "e2e": {"value": value, "unit": "sample-steps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------
# GPU arm
# ---------------------------------------------------------------------------
def _device_inputs(B, C, np, torch, inputs):
    R = len(inputs)
    d_in = torch.from_numpy(np.frombuffer(bytes(B.make_inputs(inputs)), dtype=np.uint8).copy()).cuda()
    d_out = torch.zeros(R * C.sizeof(B.sbs_output), dtype=torch.uint8, device="cuda")
    return d_in, d_out


def _red_dev(dist):
    """Device of the small max / gather tensors: the GPU under NCCL, the host under gloo."""
    return "cpu" if dist.get_backend() == "gloo" else "cuda"


def _peer_connect(ctrl, dist, world):
    """Trade the exchange buffers' IPC handles; every rank must end on the same exchange."""
    ok, why = True, ""
    try:
        handle, _ = ctrl.peer_handle()
        handles = [None] * world
        dist.all_gather_object(handles, handle)
        ctrl.peer_connect(handles=handles)
    except Exception as exc:  # noqa: BLE001
        ok, why = False, str(exc)[:80]
    oks = [None] * world
    dist.all_gather_object(oks, ok)
    if all(oks):
        return "peer-memory stores (NVLink) + stream flag waits"
    if ok:
        ctrl.peer_connect()  # disconnect
    return f"NCCL all-gather (peer exchange unavailable on some rank: {why})"


def run_sbs(args):
    import ctypes as C

    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2403_11383_b200 import binding as B
    from paper_2403_11383_b200 import build
    from paper_2403_11383_b200 import workloads as W

    rank, world, local = dist_env()
    assert world == args.gpus or world == 1, "launch N > 1 with torchrun --nproc-per-node N"
    if args.same_gpu:
        assert args.exchange == "peer", "--same-gpu checks the peer-memory path (NCCL needs distinct GPUs)"
        local = 0
    torch.cuda.set_device(local)
    if world > 1:
        if args.exchange == "nccl" and rank == 0:
            os.environ.setdefault("NCCL_DEBUG", "INFO")  # the communicator lines go to stderr
        dist.init_process_group("gloo" if args.same_gpu else "nccl",
                                device_id=None if args.same_gpu else torch.device("cuda", local))
    if rank == 0:
        build.build()
    if world > 1:
        dist.barrier()
    B.load_library()

    K = k_total(args, world)
    cfg, inputs = W.config4(K)
    nccl_id = None
    if world > 1 and not args.same_gpu:  # (NCCL rejects two ranks on one GPU; --same-gpu uses the peer path only)
        obj = [B.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        nccl_id = obj[0]
    ctrl = B.Controller(cfg, device=local, rank=rank, world=world, nccl_id=nccl_id)
    ctrl.set_reference(0, inputs[0]["xref"])
    exchange = "none (one GPU)"
    if world > 1:
        exchange = _peer_connect(ctrl, dist, world) if args.exchange == "peer" else \
            "NCCL all-gather (ncclAllGather of the rank records on the context's stream)"
        dist.barrier()
    d_in, d_out = _device_inputs(B, C, np, torch, inputs)
    stream = torch.cuda.current_stream()
    sp = stream.cuda_stream
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")  # > 126 MB L2

    def step():
        ctrl.step_device(d_in.data_ptr(), d_out.data_ptr(), sp)

    for _ in range(max(args.warmup, 3)):
        flush.zero_()
        step()
    torch.cuda.synchronize()

    # ---- timed region: device time per iteration, L2 flushed between iterations ----
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.3)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    for i in range(args.steps):
        flush.zero_()
        ev[i][0].record(stream)
        prof = i % PROFILE_EVERY == 0  # per-kernel events on a sample of the timed steps
        if prof:
            ctrl.profile(True)
        step()
        if prof:
            ctrl.profile(False)
        ev[i][1].record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ktimes = ctrl.kernel_times()
    clk = clocks.stop()
    per = [a.elapsed_time(b) for a, b in ev]  # ms
    tot = sum(per)
    r_ms, r_n = ktimes["rollout"]
    r_avg_s = (r_ms / max(r_n, 1)) * 1e-3
    rank_times = None
    if world > 1:
        t = torch.tensor([tot], dtype=torch.float64, device=_red_dev(dist))
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        tot_max = float(t.item())
        mine = torch.tensor([tot / args.steps * 1e3, r_avg_s * 1e6], dtype=torch.float64, device=_red_dev(dist))
        allr = [torch.zeros_like(mine) for _ in range(world)]
        dist.all_gather(allr, mine)
        rank_times = [{"rank": i, "us_per_step": float(x[0]), "rollout_kernel_us": float(x[1]),
                       "exchange_and_merge_us": float(x[0] - x[1])} for i, x in enumerate(allr)]
        tot = tot_max
    ms = tot / args.steps
    value = K * H / (ms * 1e-3)
    per_sorted = sorted(per)

    def pct(q):
        return 1e3 * per_sorted[min(len(per) - 1, int(q * len(per)))]

    lat = {"p5": pct(0.05), "p50": pct(0.5), "p95": pct(0.95), "p99": pct(0.99), "mean": 1e3 * ms,
           "note": "per-iteration device time, L2 flushed before each; every 10th step carries per-kernel events"}

    # ---- roofline of the dominant kernel (the fused rollout), timed live in the same region ----
    K_local = K // world
    flops = ALG_FLOP_FUSED * K_local * H
    achieved = flops / r_avg_s / 1e12
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else {}
    sm_max = float(peaks.get("sm_max_mhz", 1965.0))
    n_sm = torch.cuda.get_device_properties(local).multi_processor_count
    peak = n_sm * FP32_LANES_PER_SM * 2 * sm_max * 1e6 / 1e12
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tpath):
        traffic = json.load(open(tpath)).get("rollout_config4_bytes_per_launch")
    roof = {"bound": "alu", "achieved": achieved, "peak": peak, "unit": "TFLOP/s", "frac": achieved / peak,
            "traffic": traffic, "kernel": "sbs_rollout_kernel<4,MPPI,fused,...,model> (sampling + rollout + MPPI)",
            "kernel_us": r_avg_s * 1e6, "kernel_share_of_step": (r_avg_s * 1e3) / ms,
            "peak_basis": f"{n_sm} SM x {FP32_LANES_PER_SM} FP32 lanes x 2 x {sm_max:.0f} MHz (clocks.max.sm, "
                          "MEASURED_PEAKS.json); derived from the profiling guide's unit counts",
            "flop_per_sample_step": FLOP_BREAKDOWN, "units_per_launch": f"{K_local} samples x {H} steps",
            "traffic_note": "dram__bytes_read + dram__bytes_write of one launch (ncu --set full, profiles/)"}

    # ---- e2e: public host API (host buffers), host clock, same workload ----
    e2e = _e2e(ctrl, B, np, torch, inputs, flush, args.e2e_steps, world, dist, K)

    line = None
    extra = None
    latency = None
    if world == 1 and not args.no_other_configs:
        latency = _latency_config2(B, W, C, np, torch, flush, args)
        extra = {"config3_cem": _time_config(B, W, C, np, torch, W.config3("cem"), steps=200, warmup=10, peak=peak,
                                             label="config3: CEM K_e=1000, K=10000, gait adaptation"),
                 "config5_batched": _time_config(B, W, C, np, torch, W.config5(), steps=20, warmup=3, peak=peak,
                                                 label="config5: 4096 robots x 1024 samples, MPPI (1 GPU)"),
                 "config5_closed_loop": _time_closed_loop(B, W, C, np, torch, W.config5(), n_iter=50),
                 # the config-4 sweep below the headline size (BASELINE configs[3]: 64k-4M samples; the
                 # north star's ">= 50 % of FP32 peak at >= 1M samples")
                 "config4_sweep": {f"2^{lk}": _time_config(B, W, C, np, torch, W.config4(1 << lk), steps=20, warmup=3,
                                                           peak=peak, label=f"config4: MPPI, K=2^{lk}")
                                   for lk in (16, 18, 20, 21)}}
    elif world > 1 and not args.no_other_configs:
        extra = {"config5_robot_sharded": _config5_sharded(B, W, C, np, torch, dist, rank, world, local, flush)}
    if rank == 0:
        cpu = None
        if not args.no_cpu_baseline:
            K_s = 16384
            cv, ctimes = oracle_rate(K_s, n_steps=max(1, int(15.0 / (K_s * H * 0.6e-6))))
            cpu = {"value": cv, "unit": "sample-steps/s", "cores": 1, "kind": "oracle",
                   "sample": f"{len(ctimes)} oracle iterations of the config-4 scenario on {K_s} of its {K} samples "
                             f"({sum(ctimes):.1f} s, single thread)"}
            try:  # the same oracle on every host core (one process each), for context
                av, ncores = oracle_rate_all_cores(4096, 10)
                cpu["all_cores"] = {"value": av, "unit": "sample-steps/s", "cores": ncores,
                                    "sample": f"{ncores} processes x 10 oracle iterations of the config-4 scenario on "
                                              "4096 samples (wall clock incl. process start)"}
            except Exception as exc:  # noqa: BLE001
                cpu["all_cores"] = {"error": str(exc)[:200]}
        line = {
            "metric": METRIC, "value": value, "unit": "sample-steps/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "latency_us": lat, "higher_is_better": True,
            "scaling": args.scaling, "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": headline_config(args, world, exchange if world > 1 else None),
            "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "latency": latency, "exchange": exchange,
            "per_rank": rank_times, "other_configs": extra,
            "same_gpu_code_path_check": bool(args.same_gpu) or None,
            "gpu_launches": int(ctrl.launches_per_step() * args.steps), "clocks": clk,
        }
        print(json.dumps(line), flush=True)
    ctrl.close()
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def _e2e(ctrl, B, np, torch, inputs, flush, n, world, dist, K):
    """sbs_set_reference + sbs_step with host buffers (inputs copied up, outputs read back
    every step), host clock, max over ranks."""
    out_arr = (B.sbs_output * 1)()
    in_arr = B.make_inputs(inputs)
    xref = np.ascontiguousarray(inputs[0]["xref"], dtype=np.float32)
    for _ in range(5):
        ctrl.set_reference(0, xref)
        ctrl.step_raw(in_arr, out_arr)
    if world > 1:
        dist.barrier()
    times = []
    for _ in range(n):
        flush.zero_()
        torch.cuda.synchronize()
        t = time.perf_counter()
        ctrl.set_reference(0, xref)
        ctrl.step_raw(in_arr, out_arr)
        times.append(time.perf_counter() - t)
    e2e_s = sum(times)
    if world > 1:
        t = torch.tensor([e2e_s], dtype=torch.float64, device=_red_dev(dist))
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())
    e2e_ms = 1e3 * e2e_s / n
    import ctypes as C
    return {"value": K * H / (e2e_ms * 1e-3), "unit": "sample-steps/s",
            "h2d_bytes_per_step": C.sizeof(B.sbs_input) + xref.nbytes, "d2h_bytes_per_step": C.sizeof(B.sbs_output),
            "ms_per_step": e2e_ms, "api": "sbs_set_reference + sbs_step (host buffers, synchronous), host clock"}


def _latency_config2(B, W, C, np, torch, flush, args):
    """Config 2 (the paper's settings, K = 10,000): per-iteration device latency with the
    L2 flushed before each, and the same through sbs_set_reference + sbs_step."""
    cfg, inputs = W.config2(K_LATENCY)
    ctrl = B.Controller(cfg)
    ctrl.set_reference(0, inputs[0]["xref"])
    d_in, d_out = _device_inputs(B, C, np, torch, inputs)
    s = torch.cuda.current_stream()
    for _ in range(20):
        ctrl.step_device(d_in.data_ptr(), d_out.data_ptr(), s.cuda_stream)
    n = 1000
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(n)]
    torch.cuda.synchronize()
    for e0, e1 in ev:
        flush.zero_()
        e0.record(s)
        ctrl.step_device(d_in.data_ptr(), d_out.data_ptr(), s.cuda_stream)
        e1.record(s)
    torch.cuda.synchronize()
    us = sorted(a.elapsed_time(b) * 1e3 for a, b in ev)
    e2e = _e2e(ctrl, B, np, torch, inputs, flush, 500, 1, None, K_LATENCY)
    ctrl.close()
    mean = sum(us) / n
    return {"workload": "config2: MPPI, K=10000, H=12, dt=0.02 s, fixed trot, cmd 0.5 m/s (BASELINE.json configs[1])",
            "us_per_iteration": {"p5": us[n // 20], "p50": us[n // 2], "p95": us[19 * n // 20], "p99": us[99 * n // 100],
                                 "mean": mean},
            "value": K_LATENCY * H / (mean * 1e-6), "unit": "sample-steps/s",
            "e2e_us": e2e["ms_per_step"] * 1e3, "e2e": e2e,
            "timing": "1000 isolated iterations, L2 flushed before each, CUDA events; e2e: host clock around "
                      "sbs_set_reference + sbs_step"}


def _time_config(B, W, C, np, torch, cfg_inputs, steps, warmup, peak, label):
    """Device time per iteration of another BASELINE config (inputs resident, L2 flushed
    between iterations), with the rollout kernel's live roofline fraction."""
    cfg, inputs = cfg_inputs
    R = len(inputs)
    ctrl = B.Controller(cfg)
    for r, inp in enumerate(inputs):
        ctrl.set_reference(r, inp["xref"])
    d_in, d_out = _device_inputs(B, C, np, torch, inputs)
    stream = torch.cuda.current_stream()
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")
    for _ in range(warmup):
        ctrl.step_device(d_in.data_ptr(), d_out.data_ptr(), stream.cuda_stream)
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    for i in range(steps):
        flush.zero_()
        ev[i][0].record(stream)
        prof = i % 2 == 0
        if prof:
            ctrl.profile(True)
        ctrl.step_device(d_in.data_ptr(), d_out.data_ptr(), stream.cuda_stream)
        if prof:
            ctrl.profile(False)
        ev[i][1].record(stream)
    torch.cuda.synchronize()
    kt = ctrl.kernel_times()
    # iteration time from the steps without per-kernel events (those break the
    # programmatic-launch overlap between the kernels); kernel times from the others
    plain = [a.elapsed_time(b) for i, (a, b) in enumerate(ev) if i % 2 == 1]
    ms = sum(plain) / len(plain)
    K = cfg["n_samples"] * R
    r_ms, r_n = kt["rollout"]
    r_s = r_ms / max(r_n, 1) * 1e-3
    achieved = ALG_FLOP_FUSED * K * H / r_s / 1e12
    ctrl.close()
    return {"workload": label, "K_total": K, "steps": steps, "ms_per_step": ms,
            "timing": "L2 flushed before every step; ms_per_step over the odd steps, kernels_us from the even "
                      "steps (per-kernel CUDA events)",
            "value": K * H / (ms * 1e-3), "unit": "sample-steps/s",
            "kernels_us": {k: 1e3 * v[0] / v[1] for k, v in kt.items() if v[1]},
            "rollout_roofline": {"bound": "alu", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                                 "frac": achieved / peak}}


def _time_closed_loop(B, W, C, np, torch, cfg_inputs, n_iter):
    """Config 5 as a batched closed loop (sbs_run_loop): every control step is the MPC
    iteration for all robots plus the on-device plant / footholds / reference advance."""
    cfg, inputs = cfg_inputs
    R = len(inputs)
    ctrl = B.Controller(cfg)
    for r, inp in enumerate(inputs):
        ctrl.set_reference(r, inp["xref"])
    d_in, d_out = _device_inputs(B, C, np, torch, inputs)
    fallen = torch.zeros(R, dtype=torch.int32, device="cuda")
    lc = W.loop_config()
    s = torch.cuda.current_stream()
    ctrl.run_loop(3, d_in.data_ptr(), d_out.data_ptr(), 0, 0, fallen.data_ptr(), 0, lc, s.cuda_stream)  # warm-up
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(s)
    ctrl.run_loop(n_iter, d_in.data_ptr(), d_out.data_ptr(), 0, 0, fallen.data_ptr(), 0, lc, s.cuda_stream)
    e1.record(s)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / n_iter
    K = cfg["n_samples"] * R
    n_fallen = int(fallen.sum().item())
    ctrl.close()
    return {"workload": "config5 closed loop: 4096 robots x 1024 samples, MPPI + SRBD plant, Eq. 3 footholds, "
                        "reference rebuild per control step (sbs_run_loop, one graph per step)",
            "K_total": K, "control_steps": n_iter, "ms_per_control_step": ms,
            "value": K * H / (ms * 1e-3), "unit": "sample-steps/s",
            "robot_control_steps_per_s": R / (ms * 1e-3), "fallen": n_fallen}


def _config5_sharded(B, W, C, np, torch, dist, rank, world, local, flush, steps=20):
    """Config 5 sharded by robot (BASELINE configs[4]): rank g owns robots
    [g R/N, (g+1) R/N) through `robot_offset` (the noise counter carries the global robot
    index, so every robot draws the same samples as in one context); no collective."""
    cfg, inputs = W.config5()
    R = len(inputs)
    R_loc = R // world
    lo = rank * R_loc
    mine = inputs[lo:lo + R_loc]
    cfg = dict(cfg, n_robots=R_loc)
    ctrl = B.Controller(cfg, device=local, robot_offset=lo)
    for r, inp in enumerate(mine):
        ctrl.set_reference(r, inp["xref"])
    d_in, d_out = _device_inputs(B, C, np, torch, mine)
    s = torch.cuda.current_stream()
    for _ in range(3):
        ctrl.step_device(d_in.data_ptr(), d_out.data_ptr(), s.cuda_stream)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    dist.barrier()
    torch.cuda.synchronize()
    for e0, e1 in ev:
        flush.zero_()
        e0.record(s)
        ctrl.step_device(d_in.data_ptr(), d_out.data_ptr(), s.cuda_stream)
        e1.record(s)
    torch.cuda.synchronize()
    tot = torch.tensor([sum(a.elapsed_time(b) for a, b in ev)], dtype=torch.float64, device=_red_dev(dist))
    dist.all_reduce(tot, op=dist.ReduceOp.MAX)
    ms = float(tot.item()) / steps
    ctrl.close()
    K = cfg["n_samples"] * R
    return {"workload": f"config5: {R} robots x 1024 samples, MPPI, {R_loc} robots per GPU via robot_offset "
                        "(no collective)", "K_total": K, "ms_per_step": ms, "value": K * H / (ms * 1e-3),
            "unit": "sample-steps/s", "scaling": "strong", "timing": "max over ranks, L2 flushed before each step"}


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    return run_sbs(args)


if __name__ == "__main__":
    sys.exit(main())
