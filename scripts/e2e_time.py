"""Host-path (sbs_set_reference + sbs_step) latency at config 2."""
import os, sys, time
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2403_11383_b200 import binding as B, workloads as W
B.load_library()
cfg, inputs = W.config2()
c = B.Controller(cfg)
xref = np.ascontiguousarray(inputs[0]["xref"], dtype=np.float32)
arr = B.make_inputs(inputs)
out = (B.sbs_output * 1)()
for _ in range(50):
    c.set_reference(0, xref); c.step_raw(arr, out)
for mode in ("ref+step", "step"):
    ts = []
    for _ in range(2000):
        t = time.perf_counter()
        if mode == "ref+step":
            c.set_reference(0, xref)
        c.step_raw(arr, out)
        ts.append(time.perf_counter() - t)
    ts = np.array(ts) * 1e6
    print(f"{os.environ.get('SBS_MAPPED_OUT','1')} {mode}: mean {ts.mean():.1f} us p50 {np.median(ts):.1f} p99 {np.percentile(ts,99):.1f}  device_us {out[0].device_us:.1f}")
