"""Closed-loop control-step time for one robot (K = 10k, n_inner 1 and 8) and config 5."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
from paper_2403_11383_b200 import experiments as E, workloads as W
for inner in (1, 8):
    cfg = W.base_config(n_samples=10000, mode="mppi")
    tr, fallen, ms = E.run_episodes(cfg, [W.robot_input(cfg, 0)], E._cmd_rows(1, (0, 0, 0)), None, 4.0,
                                    dict(W.loop_config(), n_inner=inner))
    print(f"one robot, K=10k, n_inner={inner}: {1e3 * ms / tr.shape[0]:.1f} us per control step")
