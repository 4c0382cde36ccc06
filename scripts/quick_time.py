"""Quick device timing of sbs_step_device for a few configs (development aid)."""
import ctypes as C
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2403_11383_b200 import binding as B  # noqa: E402
from paper_2403_11383_b200 import build, workloads as W  # noqa: E402


def dev_io(inputs, R):
    arr = B.make_inputs(inputs)
    raw = np.frombuffer(bytes(arr), dtype=np.uint8)
    d_in = torch.from_numpy(raw.copy()).cuda()
    d_out = torch.zeros(R * C.sizeof(B.sbs_output), dtype=torch.uint8, device="cuda")
    return d_in, d_out


def time_cfg(name, cfg, inputs, steps=20, warm=5):
    R = cfg.get("n_robots", 1)
    c = B.Controller(cfg)
    for r in range(R):
        c.set_reference(r, inputs[r]["xref"])
    d_in, d_out = dev_io(inputs, R)
    s = torch.cuda.current_stream()
    for _ in range(warm):
        c.step_device(d_in.data_ptr(), d_out.data_ptr(), s.cuda_stream)
    torch.cuda.synchronize()
    c.profile(True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        c.step_device(d_in.data_ptr(), d_out.data_ptr(), s.cuda_stream)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    kt = c.kernel_times()
    c.profile(False)
    # no-profile timing
    e0.record()
    for _ in range(steps):
        c.step_device(d_in.data_ptr(), d_out.data_ptr(), s.cuda_stream)
    e1.record()
    torch.cuda.synchronize()
    ms2 = e0.elapsed_time(e1) / steps
    K = cfg["n_samples"] * R
    H = cfg["horizon"]
    ksum = {k: (v[0] / max(v[1], 1)) for k, v in kt.items() if v[1]}
    print(f"{name:>10s} K={K:>9d} H={H}: {ms2*1e3:9.1f} us/step  {K*H/(ms2*1e-3):.3e} sample-steps/s  "
          f"kernels(us)={ {k: round(v*1e3,1) for k,v in ksum.items()} }", flush=True)
    # host e2e
    arr = B.make_inputs(inputs)
    out = (B.sbs_output * R)()
    c.step_raw(arr, out)
    t = time.perf_counter()
    for _ in range(steps):
        c.step_raw(arr, out)
    t = (time.perf_counter() - t) / steps
    print(f"{'':>10s} host sbs_step e2e {t*1e6:.1f} us  device_us={out[0].device_us:.1f}", flush=True)
    c.close()


def main():
    build.build()
    time_cfg("config1", *W.config1())
    time_cfg("config2", *W.config2())
    time_cfg("config3cem", *W.config3("cem"))
    time_cfg("config3nv", *W.config3("naive"))
    for lg in (16, 18, 20, 22):
        time_cfg(f"K=2^{lg}", *W.config4(1 << lg), steps=10, warm=3)
    cfg, inputs = W.config5(R=4096, M=1024)
    time_cfg("config5", cfg, inputs, steps=10, warm=3)


if __name__ == "__main__":
    main()
