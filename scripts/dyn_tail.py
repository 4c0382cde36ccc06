"""Experiments only: where the fixed cost of a dynamic-tile iteration goes (SBS_TIMING
build, config 4).  Per CTA (%globaltimer): start, end of its tile loop, end of its node
merges; the root merge's start / end (CTA that finishes the iteration).  Printed in us
relative to the earliest CTA start, median over iterations."""
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
n_sm = torch.cuda.get_device_properties(0).multi_processor_count
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for lk in [int(a) for a in sys.argv[1:]] or (18, 20, 22):
    cfg, inputs = W.config4(1 << lk)
    c = B.Controller(cfg)
    c.set_reference(0, inputs[0]["xref"])
    d_in = torch.from_numpy(np.frombuffer(bytes(B.make_inputs(inputs)), dtype=np.uint8).copy()).cuda()
    d_out = torch.zeros(C.sizeof(B.sbs_output), dtype=torch.uint8, device="cuda")
    grid = min((1 << lk) // 128, 4 * n_sm)
    rows = []
    for it in range(25):
        flush.zero_()
        torch.cuda.synchronize()
        c.step_device(d_in.data_ptr(), d_out.data_ptr(), 0)
        torch.cuda.synchronize()
        buf = (C.c_uint64 * (1024 * 6))()
        L.sbs_debug_cta_p4(buf)
        ts = (C.c_uint64 * 32)()
        L.sbs_debug_ts_p4(ts)
        a = np.array(buf[:], dtype=np.float64).reshape(1024, 6)[:grid]
        t0 = a[:, 0].min()
        if it < 5 or a[:, 0].max() - t0 > 50e3:
            continue
        start, loop_end, merged = (a[:, 0] - t0) / 1e3, (a[:, 3] - t0) / 1e3, (a[:, 1] - t0) / 1e3
        ready, l1, up = (a[:, 2] - t0) / 1e3, (a[:, 4] - t0) / 1e3, (a[:, 5] - t0) / 1e3
        def last(v):  # latest of the slots this launch wrote (static split: none)
            v = v[(v > 0) & (v < 1e5)]
            return v.max() if v.size else np.nan
        rows.append([start.max(), loop_end.min(), np.median(loop_end), loop_end.max(), last(merged),
                     (ts[5] - t0) / 1e3, (ts[6] - t0) / 1e3, last(ready), last(l1), last(up),
                     (ts[8] - t0) / 1e3, (ts[9] - t0) / 1e3, (ts[10] - t0) / 1e3])
    m = np.median(np.array(rows), axis=0)
    print(f"K=2^{lk} grid {grid}: last CTA start {m[0]:.1f} | tile loops end min {m[1]:.1f} median {m[2]:.1f} "
          f"max {m[3]:.1f} | node merges end max {m[4]:.1f} | root merge {m[5]:.1f} -> {m[6]:.1f} us "
          f"({len(rows)} iterations)")
    print(f"    last level-1 node ready {m[7]:.1f} merged {m[8]:.1f} | last upper node merged {m[9]:.1f}"
          f" | static merge: argmin {m[10]:.1f} sums {m[11]:.1f} mean written {m[12]:.1f}")
    c.close()
