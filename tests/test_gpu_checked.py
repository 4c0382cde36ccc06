"""Memory-safety and race evidence without compute-sanitizer (closed on the GPU pool):

* the whole GPU parity suite re-run against the bounds-checked build of the library
  (SBS_CHECKED: every kernel index into a context buffer -- costs, CTA records, elite
  lists, robot outputs, contact tables -- is checked against its allocation's bound and
  traps on a violation), covering every kernel and launch shape the suite reaches;
* run-to-run bit identity of whole iterations in every mode and launch mode: the
  cross-CTA arrival counters, the dynamic-tile counter and tree-node flags (K = 2^21),
  the CEM cluster's shared-memory transactions (config 3), the producer / integrator
  named barriers, cp.async staging and programmatic dependent launch would show a race
  as a difference between repeats.
"""
import os
import subprocess
import sys

import numpy as np
import pytest

from paper_2403_11383_b200 import workloads as W

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_suite_under_bounds_checked_build():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2403_11383_b200 import build
    lib = build.build_checked()
    env = dict(os.environ, SBS_LIB_PATH=lib)
    probe = subprocess.run([sys.executable, "-c", "from paper_2403_11383_b200 import binding as b; "
                            "b.load_library(); print(b.LIB_PATH)"], cwd=ROOT, env=env, capture_output=True, text=True)
    assert probe.stdout.strip() == lib, probe.stdout + probe.stderr
    files = ["tests/test_gpu_parity.py", "tests/test_gpu_parity_r2.py", "tests/test_gpu_loop.py",
             "tests/test_gpu_fullcov.py"]
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu", "-p", "no:cacheprovider", *files],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=1800)
    tail = (r.stdout + r.stderr)[-3000:]
    assert r.returncode == 0, tail
    assert "SBS_CHECK failed" not in r.stdout + r.stderr, tail


@pytest.fixture(scope="module")
def B():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2403_11383_b200 import binding, build
    build.build()
    binding.load_library()
    return binding


@pytest.mark.parametrize("which", ["c1", "c2", "c3cem", "c3naive", "c4_64k", "c4_2m", "c5_small"])
def test_repeats_are_bit_identical(B, which):
    cfg, inputs = {"c1": W.config1, "c2": W.config2, "c3cem": lambda: W.config3("cem"),
                   "c3naive": lambda: W.config3("naive"), "c4_64k": lambda: W.config4(1 << 16),
                   "c4_2m": lambda: W.config4(1 << 21),
                   "c5_small": lambda: W.config5(R=64, M=1024)}[which]()
    st = W.initial_distribution(cfg)
    ref = None
    for rep in range(12):
        c = B.Controller(cfg)
        for r, inp in enumerate(inputs):
            c.set_reference(r, inp["xref"])
        outs = [c.step(inputs)[1] for _ in range(2)]
        got = (c.debug_costs().copy(), [[o[k].copy() for k in ("mean", "var", "u0")] for step in outs for o in step])
        c.close()
        if ref is None:
            ref = got
            continue
        np.testing.assert_array_equal(got[0], ref[0])
        for a, b in zip(got[1], ref[1]):
            for x, y in zip(a, b):
                np.testing.assert_array_equal(x, y)
