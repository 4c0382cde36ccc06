"""Experiments only: host-side phase times of sbs_step (one robot, config 2; SBS_HOST_TIMING build)."""
import ctypes as C, os, sys, time
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2403_11383_b200 import build
lib = build.build(force=True, out=os.path.join(ROOT, "paper_2403_11383_b200", "libsbs_ht.so"), defines=("SBS_HOST_TIMING",))
from paper_2403_11383_b200 import binding as B, workloads as W
L = B.load_library(lib)
L.sbs_debug_host_times.argtypes = [C.POINTER(C.c_double)]
cfg, inputs = W.config2()
c = B.Controller(cfg)
c.set_reference(0, inputs[0]["xref"])
arr = B.make_inputs(inputs)
out = (B.sbs_output * 1)()
for _ in range(200):
    c.step_raw(arr, out)
buf = (C.c_double * 8)()
L.sbs_debug_host_times(buf)
ts = []
for _ in range(2000):
    t = time.perf_counter()
    c.step_raw(arr, out)
    ts.append(time.perf_counter() - t)
L.sbs_debug_host_times(buf)
names = ["validate", "blk_ev sync", "params", "event0", "launch", "event1", "stream sync", "outputs"]
print("python-level mean %.1f us; inside sbs_step: " % (np.mean(ts) * 1e6) +
      ", ".join(f"{n} {v:.2f}" for n, v in zip(names, buf)) + f" (sum {sum(buf):.1f}); device_us {out[0].device_us:.1f}")
