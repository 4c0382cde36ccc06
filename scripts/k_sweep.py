"""Experiments only: config-4 MPPI iteration time over K = 2^16 ... 2^22 on one GPU (device
time per isolated iteration with CUDA events, L2 flushed before each, median of n) and the
fused kernel's fraction of the FP32 ALU peak with the op-count numerator (bench.py)."""
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2403_11383_b200 import binding as B  # noqa: E402
from paper_2403_11383_b200 import workloads as W  # noqa: E402

ALG_FLOP_FUSED = 886.1419270833334  # bench.py
PEAK = 148 * 128 * 2 * 1965e6


def main():
    B.load_library()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    print("| K | µs / iteration (median) | sample-steps/s | fraction of the FP32 ALU peak |")
    print("|---|---|---|---|")
    for lk in range(16, 23):
        K = 1 << lk
        cfg, inputs = W.config4(K)
        c = B.Controller(cfg)
        c.set_reference(0, inputs[0]["xref"])
        d_in = torch.from_numpy(np.frombuffer(bytes(B.make_inputs(inputs)), dtype=np.uint8).copy()).cuda()
        d_out = torch.zeros(C.sizeof(B.sbs_output), dtype=torch.uint8, device="cuda")
        s = torch.cuda.current_stream()
        reps = 50 if lk < 20 else 20
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
        for _ in range(5):
            c.step_device(d_in.data_ptr(), d_out.data_ptr(), s.cuda_stream)
        for e0, e1 in ev:
            flush.zero_()
            e0.record()
            c.step_device(d_in.data_ptr(), d_out.data_ptr(), s.cuda_stream)
            e1.record()
        torch.cuda.synchronize()
        t = float(np.median([a.elapsed_time(b) * 1e3 for a, b in ev]))
        c.close()
        rate = K * 12 / (t * 1e-6)
        print(f"| 2^{lk} | {t:.1f} | {rate:.3g} | {ALG_FLOP_FUSED * rate / PEAK:.3f} |", flush=True)


if __name__ == "__main__":
    main()
