#!/usr/bin/env python
"""Benchmark of one SBS MPC iteration (arxiv 2403.11383) on B200.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl sbs|reference]

Workload at N = 1: BASELINE.json configs[1] -- MPPI at the paper's settings,
K = 10,000 samples, H = 12, dt = 0.02 s, fixed trot.  With N > 1
(torchrun, one process per GPU) every rank owns 10,000 samples of one
K = 10,000 N MPPI iteration (weak scaling): the ranks' (min, sum w, sum w theta)
records are exchanged over peer memory (each rank's finishing CTA stores its
record into every peer's buffer over NVLink; the peers' streams wait on a flag)
with an NCCL all-gather as the fallback.

One JSON line on rank 0.  `value` = sample-steps/s (K_total H / device time
per iteration, inputs resident in HBM, L2 flushed between timed iterations);
`e2e` = the same metric through the public host API (sbs_set_reference +
sbs_step with host buffers, host clock).  `--impl reference` times the CPU
oracle (the reference arm of this tier) on a bounded sample of the same
workload.
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

K_PER_GPU = 10000
H = 12
# Algorithmic FLOPs per sample-step, frozen from the oracle's
# op-counting mode over the config-2 workload (scripts/op_count.py, 256 samples;
# tests/test_oracle_opcount.py re-derives them): the rollout + cost (a2-a4) alone,
# and the whole fused kernel (+ sampling a1: binary32 Box-Muller and theta2, + MPPI a5).
ALG_FLOP_ROLLOUT = 9343.0 / 12.0          # 778.58
ALG_FLOP_FUSED = 886.1419270833334        # rollout 778.58 + sampling 95.16 + MPPI 12.40
ALG_FLOP_PER_SAMPLE_STEP = ALG_FLOP_FUSED
# per-kernel CUDA events (for the roofline's kernel time) bracket every PROFILE_EVERY-th
# timed step, so their own cost stays out of the headline per-iteration time
PROFILE_EVERY = 10
FP32_LANES_PER_SM = 128


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10000)
    ap.add_argument("--warmup", type=int, default=50)
    ap.add_argument("--impl", default="sbs", choices=["sbs", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=500)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-other-configs", action="store_true", help="skip the configs 3/4/5 lines (ncu launch lists)")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", str(rank)))
    return rank, world, local


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
def oracle_rate(K_sample: int, n_steps: int, warmup: int = 1):
    """Time the oracle as it stands (single thread) on K_sample samples of config 2."""
    from oracle import Oracle
    from paper_2403_11383_b200 import workloads as W
    orc = Oracle()
    cfg, inputs = W.config2(K=K_sample)
    st = W.initial_distribution(cfg)
    for _ in range(warmup):
        orc.step(cfg, 0, inputs[0], st, keep=False)
    times = []
    for _ in range(n_steps):
        t = time.perf_counter()
        orc.step(cfg, 0, inputs[0], st, keep=False)
        times.append(time.perf_counter() - t)
    tot = sum(times)
    return K_sample * H * n_steps / tot, times


def _oracle_worker(args):
    K_sample, n_steps = args
    rate, times = oracle_rate(K_sample, n_steps, warmup=0)
    return K_sample * H * n_steps, sum(times)


def oracle_rate_all_cores(K_sample: int, n_steps: int):
    """The same oracle iteration run concurrently in one process per host core (each on its
    own K_sample-sample slice-sized iteration): the oracle as it stands, parallelised by the
    harness only.  Returns (sample-steps/s over the wall time, processes)."""
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
    # each step: a bounded sample of the config-2 iteration sized so the whole run takes ~1-3 minutes
    budget_s = 120.0
    per_sample_step_s = 2.0e-6
    n = max(args.steps + args.warmup, 1)
    K_s = int(max(64, min(K_PER_GPU, budget_s / (n * H * per_sample_step_s))))
    value, times = oracle_rate(K_s, args.steps, warmup=args.warmup)
    ms = 1e3 * sum(times) / len(times)
    line = {
        "impl": "reference", "metric": "sample-steps/sec and MPC-iteration latency (us) at N samples",
        "value": value, "unit": "sample-steps/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms, "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": {"workload": "config2: MPPI, K=10000 samples, H=12, dt=0.02 s, fixed trot 1.3 Hz, cmd 0.5 m/s",
                   "K_per_step": K_s, "H": H},
        "cpu_baseline": {"value": value, "unit": "sample-steps/s", "cores": 1, "kind": "oracle",
                         "sample": f"{K_s} of the 10000 samples per step (same iteration), {args.steps} steps"},
        "e2e": {"value": value, "unit": "sample-steps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------
# GPU arm
# ---------------------------------------------------------------------------
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
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    if rank == 0:
        build.build()
    if world > 1:
        dist.barrier()
    B.load_library()

    K_total = K_PER_GPU * world
    cfg, inputs = W.config2(K=K_total)
    nccl_id = None
    if world > 1:
        obj = [B.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        nccl_id = obj[0]
    ctrl = B.Controller(cfg, device=local, rank=rank, world=world, nccl_id=nccl_id)
    ctrl.set_reference(0, inputs[0]["xref"])
    exchange = "none"
    if world > 1:
        # rank records exchanged over peer memory (the finishing CTA stores into every peer's
        # buffer over NVLink; streams wait on the peers' flags); NCCL all-gather as fallback
        ok, why = True, ""
        try:
            handle, _ = ctrl.peer_handle()
            handles = [None] * world
            dist.all_gather_object(handles, handle)
            ctrl.peer_connect(handles=handles)
        except Exception as exc:  # noqa: BLE001
            ok, why = False, str(exc)[:80]
        oks = [None] * world
        dist.all_gather_object(oks, ok)  # every rank must use the same exchange
        if all(oks):
            exchange = "peer memory (NVLink stores + stream flag waits)"
        else:
            if ok:
                ctrl.peer_connect()  # disconnect
            exchange = f"NCCL all-gather (peer exchange unavailable on some rank: {why})"
        dist.barrier()
    in_arr = B.make_inputs(inputs)
    d_in = torch.from_numpy(np.frombuffer(bytes(in_arr), dtype=np.uint8).copy()).cuda()
    d_out = torch.zeros(C.sizeof(B.sbs_output), dtype=torch.uint8, device="cuda")
    stream = torch.cuda.current_stream()
    sp = stream.cuda_stream
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")  # > 126 MB L2

    def step():
        ctrl.step_device(d_in.data_ptr(), d_out.data_ptr(), sp)

    for _ in range(args.warmup):
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
    if world > 1:
        t = torch.tensor([tot], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        tot = float(t.item())
    ms = tot / args.steps
    value = K_total * H / (ms * 1e-3)
    per_sorted = sorted(per)
    def pct(q):
        return 1e3 * per_sorted[min(len(per) - 1, int(q * len(per)))]

    lat = {"p5": pct(0.05), "p50": pct(0.5), "p95": pct(0.95), "p99": pct(0.99), "mean": 1e3 * ms,
           "note": "per-iteration device time, L2 flushed before each; every 10th step carries per-kernel events"}

    # ---- roofline of the dominant kernel (rollout), timed live in the same region ----
    r_ms, r_n = ktimes["rollout"]
    r_avg_s = (r_ms / max(r_n, 1)) * 1e-3
    flops = ALG_FLOP_PER_SAMPLE_STEP * K_PER_GPU * H
    achieved = flops / r_avg_s / 1e12
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else {}
    sm_max = float(peaks.get("sm_max_mhz", 1965.0))
    n_sm = torch.cuda.get_device_properties(local).multi_processor_count
    peak = n_sm * FP32_LANES_PER_SM * 2 * sm_max * 1e6 / 1e12
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tpath):
        traffic = json.load(open(tpath)).get("rollout_config2_bytes_per_launch")
    roof = {"bound": "alu", "achieved": achieved, "peak": peak, "unit": "TFLOP/s", "frac": achieved / peak,
            "traffic": traffic, "kernel": "sbs_rollout_kernel<4,MPPI,fused>",
            "kernel_us": r_avg_s * 1e6, "kernel_share_of_step": (r_avg_s * 1e3) / ms,
            "peak_basis": f"{n_sm} SM x {FP32_LANES_PER_SM} FP32 lanes x 2 x {sm_max:.0f} MHz (clocks.max.sm)",
            "flop_per_sample_step": ALG_FLOP_PER_SAMPLE_STEP}

    # ---- e2e: public host API (host buffers), host clock ----
    out_arr = (B.sbs_output * 1)()
    xref = np.ascontiguousarray(inputs[0]["xref"], dtype=np.float32)
    for _ in range(10):
        ctrl.set_reference(0, xref)
        ctrl.step_raw(in_arr, out_arr)
    if world > 1:
        dist.barrier()
    host_times = []
    for _ in range(args.e2e_steps):
        flush.zero_()
        torch.cuda.synchronize()
        t = time.perf_counter()
        ctrl.set_reference(0, xref)
        ctrl.step_raw(in_arr, out_arr)
        host_times.append(time.perf_counter() - t)
    e2e_s = sum(host_times)
    if world > 1:
        t = torch.tensor([e2e_s], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())
    e2e_ms = 1e3 * e2e_s / args.e2e_steps
    h2d = C.sizeof(B.sbs_input) + xref.nbytes
    d2h = C.sizeof(B.sbs_output)
    e2e = {"value": K_total * H / (e2e_ms * 1e-3), "unit": "sample-steps/s", "h2d_bytes_per_step": h2d,
           "d2h_bytes_per_step": d2h, "ms_per_step": e2e_ms,
           "api": "sbs_set_reference + sbs_step (host buffers, synchronous)"}

    # ---- the other BASELINE configs on this GPU (rank 0, N = 1): where the ALU roofline is
    #      meaningful (config 4 at K = 2^22) and the CEM iteration (config 3) ----
    extra = None
    if world == 1 and not args.no_other_configs:
        extra = {"config4_K4M": _time_config(B, W, C, np, torch, W.config4(4194304), steps=20, warmup=3,
                                             peak=peak, label="config4: MPPI, K=2^22, H=12 (BASELINE configs[3], 1 GPU)"),
                 "config3_cem": _time_config(B, W, C, np, torch, W.config3("cem"), steps=200, warmup=10,
                                             peak=peak, label="config3: CEM K_e=1000, K=10000, gait adaptation"),
                 "config5_batched": _time_config(B, W, C, np, torch, W.config5(), steps=20, warmup=3, peak=peak,
                                                 label="config5: 4096 robots x 1024 samples, MPPI (1 GPU)"),
                 "config5_closed_loop": _time_closed_loop(B, W, C, np, torch, W.config5(), n_iter=50)}

    line = None
    if rank == 0:
        cpu = None
        if not args.no_cpu_baseline:
            K_s = 2000
            cv, ctimes = oracle_rate(K_s, n_steps=max(1, int(12.0 / (K_s * H * 2.3e-6))))
            cpu = {"value": cv, "unit": "sample-steps/s", "cores": 1, "kind": "oracle",
                   "sample": f"{len(ctimes)} oracle iterations of config 2 on {K_s} of its 10000 samples "
                             f"({sum(ctimes):.1f} s, single thread)"}
            try:  # the same oracle on every host core (one process each), for context
                av, ncores = oracle_rate_all_cores(2000, 150)
                cpu["all_cores"] = {"value": av, "unit": "sample-steps/s", "cores": ncores,
                                    "sample": f"{ncores} processes x 150 oracle iterations of config 2 on 2000 samples (wall clock incl. process start)"}
            except Exception as exc:  # noqa: BLE001
                cpu["all_cores"] = {"error": str(exc)[:200]}
        line = {
            "metric": "sample-steps/sec and MPC-iteration latency (us) at N samples",
            "value": value, "unit": "sample-steps/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms, "latency_us": lat, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": "config2: MPPI, K=10000 samples per GPU, H=12, dt=0.02 s, fixed trot 1.3 Hz, "
                                   "cmd 0.5 m/s (BASELINE.json configs[1])",
                       "K_total": K_total, "K_per_gpu": K_PER_GPU, "H": H, "mode": "mppi",
                       "parallelism": f"samples sharded over {world} GPU(s)" + (f", rank records by {exchange}" if world > 1 else ""),
                       "l2": "flushed between timed iterations (256 MiB memset, outside the events)"},
            "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "other_configs": extra,
            "gpu_launches": int(ctrl.launches_per_step() * args.steps), "clocks": clk,
        }
        print(json.dumps(line), flush=True)
    ctrl.close()
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def _time_config(B, W, C, np, torch, cfg_inputs, steps, warmup, peak, label):
    """Device time per iteration of another BASELINE config (inputs resident, L2 flushed
    between iterations), with the rollout kernel's live roofline fraction."""
    cfg, inputs = cfg_inputs
    R = len(inputs)
    ctrl = B.Controller(cfg)
    for r, inp in enumerate(inputs):
        ctrl.set_reference(r, inp["xref"])
    d_in = torch.from_numpy(np.frombuffer(bytes(B.make_inputs(inputs)), dtype=np.uint8).copy()).cuda()
    d_out = torch.zeros(R * C.sizeof(B.sbs_output), dtype=torch.uint8, device="cuda")
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
    achieved = ALG_FLOP_PER_SAMPLE_STEP * K * H / r_s / 1e12
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
    d_in = torch.from_numpy(np.frombuffer(bytes(B.make_inputs(inputs)), dtype=np.uint8).copy()).cuda()
    d_out = torch.zeros(R * C.sizeof(B.sbs_output), dtype=torch.uint8, device="cuda")
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


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    return run_sbs(args)


if __name__ == "__main__":
    sys.exit(main())
