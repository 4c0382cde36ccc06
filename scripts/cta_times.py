"""Experiments only: per-CTA timestamps of the rollout kernel (SBS_TIMING build):
start, sampled, rolled out, record written (globaltimer), and the rollout's SM cycles."""
import ctypes as C, os, sys
import numpy as np, torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2403_11383_b200 import build
lib = build.build(force=True, out=os.path.join(ROOT, "paper_2403_11383_b200", "libsbs_timing.so"), defines=("SBS_TIMING",))
from paper_2403_11383_b200 import binding as B, workloads as W
B.LIB_PATH = lib
L = B.load_library(lib)
L.sbs_debug_cta_p4.argtypes = [C.POINTER(C.c_uint64)]
L.sbs_debug_ts_p4.argtypes = [C.POINTER(C.c_uint64)]
L.sbs_debug_bar_p4.argtypes = [C.POINTER(C.c_uint64)]
for name, (cfg, inputs) in [("c2", W.config2()), ("c3nv", W.config3("naive"))]:
    c = B.Controller(cfg)
    c.set_reference(0, inputs[0]["xref"])
    d_in = torch.from_numpy(np.frombuffer(bytes(B.make_inputs(inputs)), dtype=np.uint8).copy()).cuda()
    d_out = torch.zeros(C.sizeof(B.sbs_output), dtype=torch.uint8, device="cuda")
    n = c.n_cta if hasattr(c, "n_cta") else 79
    acc, bars = [], []
    for it in range(30):
        c.step_device(d_in.data_ptr(), d_out.data_ptr(), 0)
        torch.cuda.synchronize()
        buf = (C.c_uint64 * (1024 * 6))()
        L.sbs_debug_cta_p4(buf)
        bb = (C.c_uint64 * 32)()
        L.sbs_debug_bar_p4(bb)
        if it >= 5:
            bars.append(np.array(bb[:], dtype=np.float64).reshape(4, 8))
        ts = (C.c_uint64 * 32)()
        L.sbs_debug_ts_p4(ts)
        a = np.array(buf[:], dtype=np.float64).reshape(1024, 6)[:n]
        t0 = a[:, 0].min()
        rel = (a[:, :4] - t0) / 1e3
        cyc = a[:, 5] - a[:, 4]
        merged = (ts[6] - t0) / 1e3
        if it >= 5:
            acc.append(np.concatenate([rel.max(0), rel.min(0), [np.median(cyc), cyc.max(), merged,
                                       int(np.argmax(rel[:, 3])), rel[int(np.argmax(rel[:, 3])), 0]]]))
    m = np.median(np.array(acc), axis=0)
    print(f"{name}: max over CTAs start {m[0]:.2f} sampled {m[1]:.2f} rolled {m[2]:.2f} rec {m[3]:.2f} | "
          f"min start {m[4]:.2f} sampled {m[5]:.2f} rolled {m[6]:.2f} rec {m[7]:.2f} | rollout cycles median {m[8]:.0f} "
          f"max {m[9]:.0f} | merged {m[10]:.2f} | last CTA {m[11]:.0f} started {m[12]:.2f}")
    print(f"{name}: integrator cycles waiting per chunk barrier (CTA 0, median over iterations, per warp):")
    print(np.median(np.array(bars), axis=0)[:, :6].astype(int))
    c.close()
