"""Table I ordering in aggregate (Naive fixed vs adaptive gait, 100 paired episodes per amplitude 10-16; the trend test)."""
import sys, os, json
sys.path.insert(0, os.getcwd())
from paper_2403_11383_b200 import binding, build, experiments as E
build.build(); binding.load_library()
tot = [0.0, 0.0]
for amp in (10.0, 12.0, 14.0, 16.0):
    r = E.table1(episodes=100, amp=amp, K=10000, inner=8, variants=[("naive", 0), ("naive", 1)])
    f, a = r["results"]
    tot[0] += f["success_pct"]; tot[1] += a["success_pct"]
    print(json.dumps({"amp": amp, "fixed": f["success_pct"], "adaptive": a["success_pct"], "f_adapt": a["mean_freq"]}), flush=True)
print(json.dumps({"aggregate_fixed": tot[0], "aggregate_adaptive": tot[1]}))
