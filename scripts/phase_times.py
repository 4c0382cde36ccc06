"""Experiments only: phase timestamps of the rollout kernel (SBS_TIMING build)."""
import ctypes as C, os, sys
import numpy as np, torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2403_11383_b200 import build
lib = build.build(force=True, out=os.path.join(ROOT, "paper_2403_11383_b200", "libsbs_timing.so"), defines=("SBS_TIMING",))
os.environ["SBS_LIB_PATH"] = lib
from paper_2403_11383_b200 import binding as B, workloads as W
B.LIB_PATH = lib
L = B.load_library(lib)
L.sbs_debug_ts_p4.argtypes = [C.POINTER(C.c_uint64)]
for name, (cfg, inputs) in [("c1", W.config1()), ("c2", W.config2()), ("c3cem", W.config3("cem")), ("c3nv", W.config3("naive"))]:
    c = B.Controller(cfg)
    c.set_reference(0, inputs[0]["xref"])
    d_in = torch.from_numpy(np.frombuffer(bytes(B.make_inputs(inputs)), dtype=np.uint8).copy()).cuda()
    d_out = torch.zeros(C.sizeof(B.sbs_output), dtype=torch.uint8, device="cuda")
    acc = []
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda") if os.environ.get("FLUSH") else None
    for it in range(30):
        if flush is not None:
            flush.zero_()
        c.step_device(d_in.data_ptr(), d_out.data_ptr(), 0)
        torch.cuda.synchronize()
        ts = (C.c_uint64 * 32)()
        L.sbs_debug_ts_p4(ts)
        t = np.array(ts[:11], dtype=np.float64)
        if it >= 5:
            acc.append((t - t[0]) / 1e3)
    a = np.median(np.array(acc), axis=0)
    print(f"{name}: start 0 | robot loaded {a[1]:.2f} | sampled {a[2]:.2f} | rolled out {a[3]:.2f} | epilogue done {a[4]:.2f} | "
          f"last CTA in {a[5]:.2f} | merged {a[6]:.2f} us | staged {a[7]:.2f} argmin {a[8]:.2f} sums {a[9]:.2f} mean {a[10]:.2f}")
    c.close()
