"""Experiments only: per-kernel CUDA-event times of the CEM iteration (config 3), warm and L2-flushed."""
import ctypes as C, os, sys
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from paper_2403_11383_b200 import binding as B, workloads as W
B.load_library(B.LIB_PATH)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
cfg, inputs = W.config3("cem")
c = B.Controller(cfg); c.set_reference(0, inputs[0]["xref"])
d_in = torch.from_numpy(np.frombuffer(bytes(B.make_inputs(inputs)), dtype=np.uint8).copy()).cuda()
d_out = torch.zeros(C.sizeof(B.sbs_output), dtype=torch.uint8, device="cuda")
for fl in (False, True):
    c.profile(True)
    for _ in range(200):
        if fl: flush.zero_()
        c.step_device(d_in.data_ptr(), d_out.data_ptr(), 0)
    torch.cuda.synchronize()
    kt = c.kernel_times(); c.profile(False)
    print(sys.argv[1], "flushed" if fl else "warm", {k: round(v[0] / max(v[1], 1) * 1e3, 2) for k, v in kt.items() if v[1]})
