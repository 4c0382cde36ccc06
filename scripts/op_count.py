"""Algorithmic FLOPs per sample-step of the fused MPC-iteration kernel, from the
oracle's op-counting mode (oracle/opcount.cpp) over the config-2 workload (SURVEY
8(d): "freeze the exact number by running the oracle in op-counting mode over the
config-2 workload"; the trot average).  Itemised: sampling (a1: binary32 noise
recipe + theta2 formation), rollout + cost (a2-a4), MPPI update (a5).  Prints one
JSON line.  Measurement aid: calls only oracle/ and the input generator."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from oracle import Oracle  # noqa: E402
from paper_2403_11383_b200 import workloads as W  # noqa: E402


def count(cfg, inp, n=256):
    o = Oracle()
    st = W.initial_distribution(cfg)
    mu_shift = o.warm_shift(cfg, st["mean"])
    H = cfg["horizon"]
    tot = dict(sample=[0, 0], rollout=[0, 0, 0], mppi=[0, 0])
    J, TH = [], []
    for k in range(1, n + 1):                  # k = 0 is the preserved elite (no draw)
        theta, fs, ts, _ = o.count_sample(cfg, mu_shift, st["var"], st["freq_idx"], 0, 0, k)
        Jk, f, t, c = o.count_rollout(cfg, inp["x0"], inp["phase"], inp["feet_cur"], inp["feet_next"],
                                      inp["xref"], theta, st["freq_idx"])
        assert np.isfinite(Jk)
        tot["sample"][0] += fs
        tot["sample"][1] += ts
        tot["rollout"][0] += f
        tot["rollout"][1] += t
        tot["rollout"][2] += c
        J.append(Jk)
        TH.append(theta)
    _, fm, tm, _ = o.count_mppi(np.array(J), np.array(TH), cfg["lambda"])
    per = lambda v: v / (n * H)  # noqa: E731
    out = dict(rollout_flop=per(tot["rollout"][0]), rollout_trans=per(tot["rollout"][1]),
               rollout_cmp=per(tot["rollout"][2]), sample_flop=per(tot["sample"][0]),
               sample_trans=per(tot["sample"][1]), mppi_flop=per(fm), mppi_trans=per(tm))
    out["fused_flop"] = out["rollout_flop"] + out["sample_flop"] + out["mppi_flop"]
    return dict(per_sample_step=out, samples=n, horizon=H)


if __name__ == "__main__":
    cfg, inputs = W.config2()
    print(json.dumps(dict(workload="config2", **count(cfg, inputs[0]))))
