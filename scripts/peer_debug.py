import ctypes as C, os, sys, time
import numpy as np, torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2403_11383_b200 import binding as B, workloads as W
L = B.load_library()
L.sbs_debug_xflags.argtypes = [C.c_void_p, C.POINTER(C.c_uint32)]
world = 2
cfg, inputs = W.config2(K=10000)
d_in = torch.from_numpy(np.frombuffer(bytes(B.make_inputs(inputs)), dtype=np.uint8).copy()).cuda()
ranks = [B.Controller(cfg, rank=g, world=world) for g in range(world)]
bases = [c.peer_handle()[1] for c in ranks]
print("bases", [hex(b) for b in bases])
for c in ranks:
    c.set_reference(0, inputs[0]["xref"]); c.peer_connect(bases=bases)
streams = [torch.cuda.Stream() for _ in ranks]
outs = [torch.zeros(C.sizeof(B.sbs_output), dtype=torch.uint8, device="cuda") for _ in ranks]
torch.cuda.synchronize()
for g, c in enumerate(ranks):
    c.step_device(d_in.data_ptr(), outs[g].data_ptr(), streams[g].cuda_stream)
t = time.time()
while time.time() - t < 10:
    if all(s.query() for s in streams): break
    time.sleep(0.01)
print("done:", [s.query() for s in streams], round(time.time() - t, 3))
for c in ranks:
    f = (C.c_uint32 * 8)(); L.sbs_debug_xflags(c.ctx, f); print("flags while waiting", list(f))
if all(s.query() for s in streams):
    for c in ranks:
        f = (C.c_uint32 * 8)(); L.sbs_debug_xflags(c.ctx, f); print("flags", list(f))
    res = [B.output_dict(B.sbs_output.from_buffer_copy(o.cpu().numpy().tobytes()), 48) for o in outs]
    print([r["mean"][:3] for r in res])
os._exit(0)
