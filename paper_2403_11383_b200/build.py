"""Build libsbs.so (the C-ABI library) in-tree with nvcc for sm_100a."""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libsbs.so")
# the same sources with device-side bounds checks (SBS_CHECK, sbs_internal.h): tests only
CHECKED_LIB = os.path.join(HERE, "libsbs_checked.so")
SOURCES = ["sbs_kernels.cu", "sbs_loop.cu", "sbs_api.cpp"]
HEADERS = ["sbs_internal.h", "sbs_noise.cuh", "sbs_robot_model.h"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-diag-suppress", "177,550", "-Xcompiler", "-fPIC,-O2,-Wall", "-cudart", "static",
         "--expt-relaxed-constexpr"]


def _inputs():
    files = [os.path.join(CSRC, f) for f in SOURCES + HEADERS]
    files.append(os.path.join(ROOT, "include", "sbs.h"))
    files.append(os.path.abspath(__file__))
    return files


def stale(out: str = LIB) -> bool:
    if not os.path.exists(out):
        return True
    t = os.path.getmtime(out)
    return any(os.path.getmtime(f) > t for f in _inputs())


def _units(only_p=None):
    """(source, extra defines, object suffix): the kernels file once per knot count and once
    for the common kernels, plus the host runtime -- compiled in parallel.  only_p: one knot
    count (experiment builds)."""
    units = [("sbs_kernels.cu", [f"SBS_TU_P={p}"], f"p{p}") for p in range(2, 9) if only_p in (None, p)]
    units.append(("sbs_kernels.cu", ["SBS_TU_COMMON"], "common"))
    units.append(("sbs_loop.cu", [], "loop"))
    units.append(("sbs_api.cpp", [], "api"))
    return units


def build(force: bool = False, verbose: bool = False, out: str = LIB, defines=(), only_p=None) -> str:
    """Compile csrc/ into `out` (default: the in-tree libsbs.so).  Experiment builds (another
    `out`) may add `defines` and restrict the knot count with `only_p`."""
    if out in (LIB, CHECKED_LIB) and not force and not stale(out):
        return out
    if out == CHECKED_LIB:
        defines = (*defines, "SBS_CHECKED")
    from concurrent.futures import ThreadPoolExecutor
    tag = "" if out == LIB else "." + os.path.basename(out)
    if only_p is not None:
        assert out != LIB, "the in-tree library carries every knot count"
        defines = (*defines, f"SBS_ONLY_P={only_p}")

    def compile_unit(u):
        src, defs, suffix = u
        obj = os.path.join(CSRC, f"{src}.{suffix}{tag}.o")
        cmd = [NVCC, *ARCH, *FLAGS, *[f"-D{d}" for d in (*defines, *defs)], "-I", os.path.join(ROOT, "include"),
               "-c", os.path.join(CSRC, src), "-o", obj]
        if verbose and src.endswith(".cu"):
            cmd += ["-Xptxas", "-v"]
        subprocess.check_call(cmd)
        return obj

    with ThreadPoolExecutor(max_workers=min(10, os.cpu_count() or 4)) as ex:
        objs = list(ex.map(compile_unit, _units(only_p)))
    tmp = out + f".tmp{os.getpid()}"
    subprocess.check_call([NVCC, *ARCH, "-shared", "-cudart", "static", "-o", tmp, *objs, "-ldl"])
    os.replace(tmp, out)
    return out


def build_checked(force: bool = False) -> str:
    """The bounds-checked variant of the library (tests: tests/test_gpu_checked.py)."""
    return build(force=force, out=CHECKED_LIB)


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
    if "--checked" in sys.argv:
        print(build_checked(force="--force" in sys.argv))
