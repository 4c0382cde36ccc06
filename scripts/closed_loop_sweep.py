"""Parameter sweep of the desk-scale closed loop (batched episodes on the device).
usage: closed_loop_sweep.py AMPS SIGS 'JSON list of [mode, adapt, lambda, n_inner, K, n_elite]' [seconds] [cmd_vx]"""
import json, os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2403_11383_b200.experiments import run_episodes, _cmd_rows
from paper_2403_11383_b200 import workloads as W

E = 50
seconds = float(sys.argv[4]) if len(sys.argv) > 4 else 10.0
vx = float(sys.argv[5]) if len(sys.argv) > 5 else 0.5
variants = json.loads(sys.argv[3])
for amp in [float(a) for a in sys.argv[1].split(",")]:
    for sig in [float(a) for a in sys.argv[2].split(",")]:
        for mode, adapt, lam, inner, K, ke in variants:
            cfg = W.base_config(n_samples=K, mode=mode, gait_adapt=adapt, n_robots=E, n_elite=ke,
                                sigma=[8.0 * sig, 8.0 * sig, 15.0 * sig], **{"lambda": lam})
            cmdv = (vx, 0.0, 0.0)
            inputs = [W.robot_input(cfg, e, cmd=cmdv) for e in range(E)]
            n = int(round(seconds / cfg["dt"]))
            rng = np.random.default_rng(1234)
            nh = 100
            draws = rng.uniform(-amp, amp, size=(n // nh + 1, E, 6)).astype(np.float32)
            w = np.repeat(draws, nh, axis=0)[:n]
            lc = dict(W.loop_config(), n_inner=inner)
            tr, fallen, ms = run_episodes(cfg, inputs, _cmd_rows(E, cmdv), w, seconds, lc=lc)
            alive = tr[:, :, 14] == 0
            verr = np.linalg.norm(tr[:, :, 3:5] - np.array(cmdv[:2]), axis=2)
            print(json.dumps(dict(amp=amp, sig=sig, mode=mode, adapt=adapt, lam=lam, inner=inner, K=K,
                                  success=round(100.0 * float(np.mean(fallen == 0)), 1),
                                  verr=round(float(np.mean(verr[alive])), 3) if alive.any() else None,
                                  freq=round(float(np.mean(tr[:, :, 12][alive])), 3) if alive.any() else None,
                                  jmin=round(float(np.median(tr[:, :, 13][alive])), 3) if alive.any() else None,
                                  ms=round(ms, 1))), flush=True)
