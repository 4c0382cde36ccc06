"""Experiments only: build variant libraries (one knot count, extra defines) next to the
in-tree one, e.g. python scripts/exp_build.py mb5:SBS_ROLLOUT_MIN_BLOCKS=5 mb6:SBS_ROLLOUT_MIN_BLOCKS=6"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2403_11383_b200 import build  # noqa: E402

for spec in sys.argv[1:]:
    tag, _, defs = spec.partition(":")
    out = os.path.join(build.HERE, f"libsbs_{tag}.so")
    print(build.build(force=True, out=out, defines=tuple(d for d in defs.split(",") if d), only_p=4))
