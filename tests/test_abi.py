"""CPU checks of the boundary: libsbs.so builds, loads without a GPU, exports
every function include/sbs.h declares, and its struct layouts match the
Python binding.  No compute calls (no GPU here)."""
import ctypes as C
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    from paper_2403_11383_b200 import build
    build.build()
    from paper_2403_11383_b200 import binding
    return binding.load_library()


def _declared():
    src = open(os.path.join(ROOT, "include", "sbs.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(sbs_[a-z_0-9]+)\s*\(", src)))


def test_exports_every_declared_symbol(lib):
    names = _declared()
    assert len(names) >= 25
    out = subprocess.check_output(["nm", "-D", "--defined-only", os.path.join(ROOT, "paper_2403_11383_b200", "libsbs.so")]).decode()
    exported = set(l.split()[-1] for l in out.splitlines() if " T " in l)
    missing = [n for n in names if n not in exported]
    assert not missing, missing
    for n in names:
        getattr(lib, n)


def test_struct_layouts(lib):
    from paper_2403_11383_b200 import binding as B
    assert lib.sbs_sizeof_config() == C.sizeof(B.sbs_config)
    assert lib.sbs_sizeof_input() == C.sizeof(B.sbs_input) == 160
    assert lib.sbs_sizeof_output() == C.sizeof(B.sbs_output)
    assert lib.sbs_version() == 1


def test_status_strings_and_errors_without_gpu(lib):
    assert lib.sbs_status_str(0) == b"SBS_OK"
    assert lib.sbs_status_str(-2) == b"SBS_ERR_SINGULAR"
    # invalid configs are rejected before any device call
    from paper_2403_11383_b200 import binding as B
    from paper_2403_11383_b200 import workloads as W
    cfg = W.base_config()
    for bad in [dict(mass=-1.0), dict(knots=9), dict(horizon=0), dict(duty_factor=1.5),
                dict(freq_hz=[2.0, 1.3]), dict(lambda_=0.0), dict(mode="cem", n_elite=0)]:
        c = dict(cfg)
        if "lambda_" in bad:
            c["lambda"] = bad.pop("lambda_")
        c.update(bad)
        cc = B.make_config(c)
        ctx = C.c_void_p()
        assert lib.sbs_create(C.byref(cc), C.byref(ctx)) == -1
        assert lib.sbs_last_error(None)


def test_sm100a_cubin_and_no_fallback():
    so = os.path.join(ROOT, "paper_2403_11383_b200", "libsbs.so")
    out = subprocess.check_output(["/usr/local/cuda/bin/cuobjdump", "--list-elf", so]).decode()
    assert "sm_100a" in out
    # the product package never imports the oracle
    pkg = os.path.join(ROOT, "paper_2403_11383_b200")
    for f in os.listdir(pkg):
        if f.endswith(".py"):
            txt = open(os.path.join(pkg, f)).read()
            assert "from oracle" not in txt and "import oracle" not in txt, f


def test_sample_count_limit(lib):
    """n_samples is capped at 2^24 (the finite / diverged counts ride in binary32 fields)."""
    from paper_2403_11383_b200 import binding as B
    from paper_2403_11383_b200 import workloads as W
    cc = B.make_config(W.base_config(n_samples=(1 << 24) + 1))
    ctx = C.c_void_p()
    assert lib.sbs_create(C.byref(cc), C.byref(ctx)) == -1
    assert b"2^24" in lib.sbs_last_error(None)
