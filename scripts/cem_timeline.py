"""Experiments only: cross-kernel %globaltimer timeline of a CEM iteration (rollout CTA 0,
select, elite; SBS_TIMING build), warm and after an L2 flush.  SBS_TIMING_LIB: prebuilt lib."""
import ctypes as C, os, sys
import numpy as np, torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
lib = os.environ.get("SBS_TIMING_LIB")
if not lib:
    from paper_2403_11383_b200 import build
    lib = build.build(force=True, out=os.path.join(ROOT, "paper_2403_11383_b200", "libsbs_timing.so"),
                      defines=("SBS_TIMING",))
from paper_2403_11383_b200 import binding as B, workloads as W
L = B.load_library(lib)
for n in ("sbs_debug_ts_common", "sbs_debug_ts_p4"):
    getattr(L, n).argtypes = [C.POINTER(C.c_uint64)]
cfg, inputs = W.config3("cem")
c = B.Controller(cfg)
c.set_reference(0, inputs[0]["xref"])
d_in = torch.from_numpy(np.frombuffer(bytes(B.make_inputs(inputs)), dtype=np.uint8).copy()).cuda()
d_out = torch.zeros(C.sizeof(B.sbs_output), dtype=torch.uint8, device="cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for fl in (False, True):
    acc = []
    for it in range(40):
        if fl:
            flush.zero_()
            if os.environ.get("SLEEP_CYC"):
                torch.cuda._sleep(int(os.environ["SLEEP_CYC"]))
        e0.record()
        c.step_device(d_in.data_ptr(), d_out.data_ptr(), 0)
        e1.record()
        torch.cuda.synchronize()
        a = (C.c_uint64 * 32)(); L.sbs_debug_ts_p4(a)
        b = (C.c_uint64 * 32)(); L.sbs_debug_ts_common(b)
        t0 = a[0]
        if os.environ.get("SBS_CEM_CLUSTER", "1") != "0":  # one-launch path: slots 16.. of the P TU
            row = [(a[4] - t0), (a[16] - t0), (a[16 + 2] - t0), (a[16 + 3] - t0), (a[16 + 4] - t0), (a[16 + 5] - t0),
                   (a[16 + 7] - t0), (a[24] - t0), (a[22] - t0), (a[26] - t0), (a[30] - t0), (a[29] - t0),
                   (a[28] - t0), e0.elapsed_time(e1) * 1e3, (a[25] - t0), (a[17 + 0] - t0)]
            if it >= 5:
                acc.append(np.array(row, dtype=np.float64))
            continue
        row = [(a[4] - t0), (b[0] - t0), (b[6] - t0), (a[11] - t0), (a[12] - t0), e0.elapsed_time(e1) * 1e3] + \
              [(b[i] - b[0]) for i in range(1, 9)]
        if it >= 5:
            acc.append(np.array(row, dtype=np.float64))
    m = np.median(np.array(acc), axis=0)
    if os.environ.get("SBS_CEM_CLUSTER", "1") != "0":
        m[:13] /= 1e3
        print(f"{sys.argv[1] if len(sys.argv) > 1 else ''} {'flushed' if fl else 'warm'} cluster: rollout CTA0 record {m[0]:.2f} | "
              f"released {m[1]:.2f} first load {m[15] / 1e3:.2f} keys {m[2]:.2f} pass1-2 {m[3]:.2f} pass3 {m[4]:.2f} scan {m[5]:.2f} compact {m[6]:.2f} "
              f"selected {m[7]:.2f} | rank1 elites in {m[8]:.2f} | regen done rank0 {m[9]:.2f} rank1 {m[10]:.2f} | "
              f"records in {m[11]:.2f} summed {m[14] / 1e3:.2f} | end {m[12]:.2f} | events {m[13]:.2f} us")
        continue
    m[:5] /= 1e3
    m[6:] /= 1e3
    print(f"{sys.argv[1] if len(sys.argv) > 1 else ''} {'flushed' if fl else 'warm'}: rollout CTA0 start 0 | CTA0 record {m[0]:.2f} | "
          f"select released {m[1]:.2f} end {m[2]:.2f} (merge {m[6]:.2f} keys {m[7]:.2f} pass1 {m[8]:.2f} pass2 {m[9]:.2f} scans {m[10]:.2f} writes {m[12]:.2f} synced {m[13]:.2f} end {m[11]:.2f}) | elite released {m[3]:.2f} end {m[4]:.2f} | events {m[5]:.2f} us")
