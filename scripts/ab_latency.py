"""Experiments only: per-iteration device latency of sbs_step_device (median over many
single iterations, CUDA events around each, optional L2 flush before each), for A/B
comparisons of two builds: SBS_LIB_PATH=<lib> python scripts/ab_latency.py [tag]."""
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2403_11383_b200 import binding as B  # noqa: E402
from paper_2403_11383_b200 import workloads as W  # noqa: E402


def lat(cfg, inputs, reps=400, flush=None):
    R = cfg.get("n_robots", 1)
    c = B.Controller(cfg)
    for r in range(R):
        c.set_reference(r, inputs[r]["xref"])
    d_in = torch.from_numpy(np.frombuffer(bytes(B.make_inputs(inputs)), dtype=np.uint8).copy()).cuda()
    d_out = torch.zeros(R * C.sizeof(B.sbs_output), dtype=torch.uint8, device="cuda")
    s = torch.cuda.current_stream()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
    for _ in range(10):
        c.step_device(d_in.data_ptr(), d_out.data_ptr(), s.cuda_stream)
    for e0, e1 in ev:
        if flush is not None:
            flush.zero_()
        e0.record()
        c.step_device(d_in.data_ptr(), d_out.data_ptr(), s.cuda_stream)
        e1.record()
    torch.cuda.synchronize()
    t = np.array([a.elapsed_time(b) * 1e3 for a, b in ev])
    c.close()
    return float(np.median(t)), float(np.mean(t))


def main():
    tag = sys.argv[1] if len(sys.argv) > 1 else os.path.basename(B.LIB_PATH)
    B.load_library(B.LIB_PATH)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    rows = []
    for name, (cfg, inputs) in [("c1", W.config1()), ("c2", W.config2()), ("c3cem", W.config3("cem")),
                                ("c3nv", W.config3("naive"))]:
        w = lat(cfg, inputs)
        f = lat(cfg, inputs, flush=flush)
        rows.append(f"{name} warm {w[0]:.2f} (mean {w[1]:.2f}) flushed {f[0]:.2f} (mean {f[1]:.2f})")
    if os.environ.get("AB_BIG"):
        for name, (cfg, inputs) in [("K4M", W.config4(1 << 22)), ("c5", W.config5(R=4096, M=1024))]:
            w = lat(cfg, inputs, reps=20)
            rows.append(f"{name} {w[0]:.1f} (mean {w[1]:.1f})")
    print(f"[{tag}] " + " | ".join(rows), flush=True)


if __name__ == "__main__":
    main()
