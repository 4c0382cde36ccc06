"""Run a few sbs_step_device iterations of one workload (for ncu captures)."""
import argparse
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2403_11383_b200 import binding as B  # noqa: E402
from paper_2403_11383_b200 import build, workloads as W  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="c2", choices=["c1", "c2", "c3cem", "c3naive", "c4", "c5"])
ap.add_argument("--K", type=int, default=1 << 22)
ap.add_argument("--steps", type=int, default=6)
a = ap.parse_args()
build.build()
cfg, inputs = {"c1": W.config1, "c2": W.config2, "c3cem": lambda: W.config3("cem"),
               "c3naive": lambda: W.config3("naive"), "c4": lambda: W.config4(a.K),
               "c5": W.config5}[a.workload]()
R = cfg.get("n_robots", 1)
c = B.Controller(cfg)
for r in range(R):
    c.set_reference(r, inputs[r]["xref"])
arr = B.make_inputs(inputs)
d_in = torch.from_numpy(np.frombuffer(bytes(arr), dtype=np.uint8).copy()).cuda()
d_out = torch.zeros(R * C.sizeof(B.sbs_output), dtype=torch.uint8, device="cuda")
for _ in range(a.steps):
    c.step_device(d_in.data_ptr(), d_out.data_ptr(), torch.cuda.current_stream().cuda_stream)
torch.cuda.synchronize()
print("done", a.workload, cfg["n_samples"] * R)
