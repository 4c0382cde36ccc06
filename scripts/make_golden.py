"""Write tests/golden/config1_oracle.json: a regression fixture of the ORACLE's
config-1 iteration (BASELINE.json configs[0]).  Calls only oracle/ and the
seeded workload generator; never the CUDA path."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import Oracle  # noqa: E402
from paper_2403_11383_b200 import workloads as W  # noqa: E402


def main():
    o = Oracle()
    cfg, inputs = W.config1()
    st = W.initial_distribution(cfg)
    steps = []
    for it in range(3):
        r = o.step(cfg, 0, inputs[0], st)
        steps.append(dict(status=r.status, J=[float(v) for v in r.J], mean=[float(v) for v in r.mean],
                          u0=[float(v) for v in r.u0], freq_idx=r.freq_idx, j_min=r.j_min, ess=r.ess,
                          z_bits_row1=[int(v) for v in r.z[1].view("uint32")]))
    out = dict(source="scripts/make_golden.py (oracle only): 3 iterations of config 1 from the initial "
                      "distribution; regression fixture, not an independent pin",
               steps=steps)
    path = os.path.join(ROOT, "tests", "golden", "config1_oracle.json")
    json.dump(out, open(path, "w"), indent=0)
    print("wrote", path)


if __name__ == "__main__":
    main()
