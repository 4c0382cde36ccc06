"""Desk-scale closed-loop experiments on the device: every episode is a
robot of one batched context, stepped by sbs_run_loop (MPC iteration + SRBD plant +
Eq. 3 footholds + reference rebuild, all on the GPU).

  hover  : zero command, no disturbance, 10 s
  fig4   : Naive with gait adaptation, 0.1 m/s lateral command, 40 N lateral push for
           3 s: the step frequency should rise during the push and return
  table1 : E episodes of random CoM wrenches within +/- A N / Nm, redrawn every 2 s
           (P:375), fixed vs adaptive gait: success rate and mean cost (Table I)

Every control step runs n_inner SBS iterations on the same state (Alg. 1 "multiple
times"; L34) before the plant advances.

Host-side harness only (scenario set-up and statistics over the device trace);
every step of the loop runs in the library's kernels.

usage: python -m paper_2403_11383_b200.experiments [hover|fig4|table1|all] [--episodes E] [--amp A] [--K K]
       [--inner N]
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import sys
import time

import numpy as np
import torch

from . import binding as B
from . import workloads as W


def run_episodes(cfg, inputs, cmd, wrench, seconds, lc=None):
    """Run R = len(inputs) episodes for `seconds`; wrench [n][R][6] (numpy) or None.
    Returns trace [n][R][16] (numpy), fallen [R], device ms."""
    B.load_library()
    R = len(inputs)
    n = int(round(seconds / cfg["dt"]))
    lc = lc or W.loop_config()
    c = B.Controller(cfg)
    for r, inp in enumerate(inputs):
        c.set_reference(r, inp["xref"])
    d_in = torch.from_numpy(np.frombuffer(bytes(B.make_inputs(inputs)), dtype=np.uint8).copy()).cuda()
    d_out = torch.zeros(R * C.sizeof(B.sbs_output), dtype=torch.uint8, device="cuda")
    d_cmd = torch.from_numpy(np.asarray(cmd, dtype=np.float32).reshape(R, 4)).cuda()
    d_w = torch.from_numpy(np.asarray(wrench, dtype=np.float32)).cuda() if wrench is not None else None
    fallen = torch.zeros(R, dtype=torch.int32, device="cuda")
    trace = torch.zeros((n, R, B.SBS_TRACE_FLOATS), dtype=torch.float32, device="cuda")
    s = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    c.run_loop(n, d_in.data_ptr(), d_out.data_ptr(), d_cmd.data_ptr(), d_w.data_ptr() if d_w is not None else 0,
               fallen.data_ptr(), trace.data_ptr(), lc, s.cuda_stream)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    c.close()
    return trace.cpu().numpy(), fallen.cpu().numpy(), ms


def _cmd_rows(R, v):
    cmd = np.zeros((R, 4), dtype=np.float32)
    cmd[:, :3] = v
    return cmd


def hover(K=10000, inner=8):
    cfg = W.base_config(n_samples=K, mode="mppi")
    inputs = [W.robot_input(cfg, 0)]
    tr, fallen, ms = run_episodes(cfg, inputs, _cmd_rows(1, (0, 0, 0)), None, 10.0, dict(W.loop_config(), n_inner=inner))
    verr = np.linalg.norm(tr[:, 0, 3:5], axis=1)
    return dict(scenario="hover", K=K, inner=inner, fallen=int(fallen[0]), mean_vel_err=float(verr.mean()),
                z_min=float(tr[:, 0, 2].min()), z_max=float(tr[:, 0, 2].max()), device_ms=ms,
                us_per_iter=1e3 * ms / tr.shape[0])


def fig4(K=10000, push=40.0, mode="naive", adapt=1, t0=2.0, t1=5.0, seconds=8.0, inner=8):
    cfg = W.base_config(n_samples=K, mode=mode, n_elite=1 if mode != "cem" else K // 10, gait_adapt=adapt)
    cmdv = (0.0, 0.1, 0.0)
    inputs = [W.robot_input(cfg, 0, cmd=cmdv)]
    n = int(round(seconds / cfg["dt"]))
    w = np.zeros((n, 1, 6), dtype=np.float32)
    i0, i1 = int(round(t0 / cfg["dt"])), int(round(t1 / cfg["dt"]))
    w[i0:i1, 0, 1] = push                                   # lateral (world y) force at the CoM
    tr, fallen, ms = run_episodes(cfg, inputs, _cmd_rows(1, cmdv), w, seconds, dict(W.loop_config(), n_inner=inner))
    f = tr[:, 0, 12]
    win = int(round(0.5 / cfg["dt"]))
    prof = [float(f[i:i + win].mean()) for i in range(0, n, win)]
    return dict(scenario="fig4", mode=mode, adapt=adapt, K=K, inner=inner, push_N=push, fallen=int(fallen[0]),
                f_before=float(f[:i0].mean()), f_push=float(f[i0:i1].mean()),
                f_after=float(f[i1 + int(1.0 / cfg["dt"]):].mean()), f_profile_0p5s=prof,
                y_max=float(np.abs(tr[:, 0, 1]).max()), device_ms=ms)


def table1(episodes=50, amp=12.0, K=10000, seconds=10.0, hold=2.0, variants=None, inner=8):
    variants = variants or [("naive", 0), ("naive", 1), ("mppi", 0)]
    out = []
    for mode, adapt in variants:
        cfg = W.base_config(n_samples=K, mode=mode, n_elite=1, gait_adapt=adapt, n_robots=episodes)
        cmdv = (0.5, 0.0, 0.0)
        inputs = [W.robot_input(cfg, e, cmd=cmdv) for e in range(episodes)]
        n = int(round(seconds / cfg["dt"]))
        rng = np.random.default_rng(1234)                   # paired across variants
        nh = int(round(hold / cfg["dt"]))
        draws = rng.uniform(-amp, amp, size=(n // nh + 1, episodes, 6)).astype(np.float32)
        w = np.repeat(draws, nh, axis=0)[:n]
        tr, fallen, ms = run_episodes(cfg, inputs, _cmd_rows(episodes, cmdv), w, seconds,
                                      dict(W.loop_config(), n_inner=inner))
        alive = tr[:, :, 14] == 0
        jm = tr[:, :, 13]
        mean_cost = float(np.mean(jm[alive & np.isfinite(jm)])) if alive.any() else float("nan")
        verr = np.linalg.norm(tr[:, :, 3:5] - np.array(cmdv[:2]), axis=2)
        out.append(dict(mode=mode, adapt=adapt, success_pct=100.0 * float(np.mean(fallen == 0)),
                        mean_cost=mean_cost, mean_vel_err=float(np.mean(verr[alive])) if alive.any() else None,
                        mean_freq=float(np.mean(tr[:, :, 12][alive])) if alive.any() else None,
                        device_ms=ms, us_per_iter=1e3 * ms / n))
    return dict(scenario="table1", episodes=episodes, amp=amp, K=K, inner=inner, seconds=seconds, results=out)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("which", nargs="?", default="all")
    ap.add_argument("--episodes", type=int, default=50)
    ap.add_argument("--amp", type=float, default=12.0)
    ap.add_argument("--inner", type=int, default=8)
    ap.add_argument("--K", type=int, default=10000)
    ap.add_argument("--push", type=float, default=40.0)
    a = ap.parse_args()
    t = time.time()
    res = []
    if a.which in ("hover", "all"):
        res.append(hover(a.K, a.inner))
    if a.which in ("fig4", "all"):
        res.append(fig4(a.K, a.push, inner=a.inner))
        res.append(fig4(a.K, a.push, adapt=0, inner=a.inner))
    if a.which in ("table1", "all"):
        res.append(table1(a.episodes, a.amp, a.K, inner=a.inner))
    for r in res:
        print(json.dumps(r))
    print(f"# wall {time.time() - t:.1f} s", file=sys.stderr)


if __name__ == "__main__":
    main()
