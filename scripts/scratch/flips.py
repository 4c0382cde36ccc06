import sys, os, math
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
from oracle import Oracle
from paper_2403_11383_b200 import binding as B, build, workloads as W
build.build(); B.load_library()
orc = Oracle()
for pitch, wy in [(1.3, 6.0), (1.45, 1.5), (1.5, 1.0)]:
    cfg, inputs = W.config3("cem", K=3000)
    cfg = dict(cfg, n_elite=2500)
    inp = dict(inputs[0]); x0 = inp["x0"].copy(); x0[7] = W.f32(pitch); x0[10] = W.f32(wy); inp["x0"] = x0
    st = W.initial_distribution(cfg)
    c = B.Controller(cfg); c.set_reference(0, inp["xref"]); c.set_distribution(0, st["mean"], st["var"], 0)
    ro = orc.step(cfg, 0, inp, dict(st))
    c.step([inp])
    Jg = c.debug_costs()[0].astype(np.float64)
    flip = np.nonzero(np.isfinite(Jg) != np.isfinite(ro.J))[0]
    print("case", pitch, wy, "finite orc", np.isfinite(ro.J).sum(), "gpu", np.isfinite(Jg).sum(), "flips", flip.size)
    mu_s = orc.warm_shift(cfg, st["mean"])
    for k in flip[:6]:
        th, _, f = orc.sample(cfg, mu_s, st["var"], 0, 0, 0, int(k))
        _, tr = orc.rollout(cfg, inp["x0"], inp["phase"], inp["feet_cur"], inp["feet_next"], inp["xref"], th, f, traj=True)
        print("  k", k, "Jg", Jg[k], "Jo", ro.J[k], "max|pitch|", np.nanmax(np.abs(tr[:, 7])), "max|x|", np.nanmax(np.abs(tr)), "steps finite", np.isfinite(tr).all(1).sum())
