"""Experiments only: phase timestamps of the CEM select kernel (SBS_TIMING build)."""
import ctypes as C, os, sys
import numpy as np, torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2403_11383_b200 import build
lib = build.build(force=True, out=os.path.join(ROOT, "paper_2403_11383_b200", "libsbs_timing.so"), defines=("SBS_TIMING",))
from paper_2403_11383_b200 import binding as B, workloads as W
L = B.load_library(lib)
L.sbs_debug_ts_common.argtypes = [C.POINTER(C.c_uint64)]
cfg, inputs = W.config3("cem")
c = B.Controller(cfg)
c.set_reference(0, inputs[0]["xref"])
d_in = torch.from_numpy(np.frombuffer(bytes(B.make_inputs(inputs)), dtype=np.uint8).copy()).cuda()
d_out = torch.zeros(C.sizeof(B.sbs_output), dtype=torch.uint8, device="cuda")
acc = []
for it in range(30):
    c.step_device(d_in.data_ptr(), d_out.data_ptr(), 0)
    torch.cuda.synchronize()
    ts = (C.c_uint64 * 32)()
    L.sbs_debug_ts_common(ts)
    t = np.array(ts[:7], dtype=np.float64)
    if it >= 5:
        acc.append((t - t[0]) / 1e3)
a = np.median(np.array(acc), axis=0)
print("select: start 0 | merge_diag %.2f | keys %.2f | pass1 %.2f | pass2 %.2f | scans %.2f | end %.2f us" % tuple(a[1:7]))
