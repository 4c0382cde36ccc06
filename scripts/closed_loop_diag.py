"""Diagnostics of the closed loop: per-iteration outputs (ESS, J_min) for a few settings."""
import ctypes as C, json, os, sys
import numpy as np, torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2403_11383_b200 import binding as B, workloads as W
B.load_library()

def run(cfg, inp, cmdv, n, push=None):
    lc = W.loop_config()
    c = B.Controller(cfg)
    c.set_reference(0, inp["xref"])
    d_in = torch.from_numpy(np.frombuffer(bytes(B.make_inputs([inp])), dtype=np.uint8).copy()).cuda()
    d_out = torch.zeros(C.sizeof(B.sbs_output), dtype=torch.uint8, device="cuda")
    cmd = torch.tensor([[*cmdv, 0.0]], dtype=torch.float32, device="cuda")
    fallen = torch.zeros(1, dtype=torch.int32, device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    rows = []
    for i in range(n):
        w = torch.zeros((1, 6), dtype=torch.float32, device="cuda")
        if push is not None and push[0] <= i < push[1]:
            w[0, 1] = push[2]
        c.step_device(d_in.data_ptr(), d_out.data_ptr(), s)
        c.advance(d_in.data_ptr(), d_out.data_ptr(), cmd.data_ptr(), w.data_ptr(), fallen.data_ptr(), lc, s)
        o = B.output_dict(B.sbs_output.from_buffer_copy(d_out.cpu().numpy().tobytes()), 48)
        x = B.sbs_input.from_buffer_copy(d_in.cpu().numpy().tobytes())
        rows.append([*x.x0, o["j_min"], o["j_mean"], o["ess"], o["freq_hz"], int(fallen.item()),
                     *o["u0"]])
    c.close()
    return np.array(rows)

def summary(tag, R, cmdv):
    v = R[:, 3:5] - np.array(cmdv[:2])
    print(json.dumps(dict(tag=tag, fallen_at=int(np.argmax(R[:, 16])) if R[:, 16].any() else None,
        vel_err=float(np.linalg.norm(v, axis=1).mean()), z=[float(R[:, 2].min()), float(R[:, 2].max())],
        roll=float(np.abs(R[:, 6]).max()), pitch=float(np.abs(R[:, 7]).max()),
        jmin=float(np.median(R[:, 12])), jmean=float(np.median(R[:, 13])), ess=float(np.median(R[:, 14])),
        freq=float(R[:, 15].mean()), fz_sum=float(np.mean(R[:, 17:29][:, 2::3].sum(1))))))

n = int(sys.argv[1]) if len(sys.argv) > 1 else 200
for lam in (1.0, 0.1, 0.01):
    cfg = W.base_config(n_samples=10000, mode="mppi", **{"lambda": lam})
    inp = W.robot_input(cfg, 0)
    summary(f"hover mppi lambda={lam}", run(cfg, inp, (0, 0, 0), n), (0, 0, 0))
cfg = W.base_config(n_samples=10000, mode="naive")
summary("hover naive", run(cfg, W.robot_input(cfg, 0), (0, 0, 0), n), (0, 0, 0))
for lam in (1.0, 0.01):
    cfg = W.base_config(n_samples=10000, mode="mppi", **{"lambda": lam})
    summary(f"walk0.5 mppi lambda={lam}", run(cfg, W.robot_input(cfg, 0, cmd=(0.5, 0, 0)), (0.5, 0, 0), n), (0.5, 0, 0))
cfg = W.base_config(n_samples=10000, mode="naive", gait_adapt=1)
summary("push naive adapt", run(cfg, W.robot_input(cfg, 0, cmd=(0, 0.1, 0)), (0, 0.1, 0), n, push=(50, 125, 40.0)), (0, 0.1, 0))
cfg = W.base_config(n_samples=10000, mode="cem", n_elite=1000, gait_adapt=1)
summary("push cem adapt", run(cfg, W.robot_input(cfg, 0, cmd=(0, 0.1, 0)), (0, 0.1, 0), n, push=(50, 125, 40.0)), (0, 0.1, 0))
