"""Summarise ncu outputs into profiles/: a launch list (--metrics gpu__time_duration)
and the key counters of a --set full capture.  Usage:
  python scripts/ncu_summary.py launches <launches.csv> <out.md>
  python scripts/ncu_summary.py full <report.ncu-rep> <out.md> <K_samples> <H>
"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

KEYS = [
    "gpu__time_duration.sum", "sm__cycles_elapsed.avg.per_second", "launch__grid_size", "launch__block_size",
    "launch__registers_per_thread", "launch__occupancy_limit_registers", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed.avg.per_cycle_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "inst_executed", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "smsp__sass_thread_inst_executed_op_ffma_pred_on.sum.per_cycle_elapsed",
    "smsp__sass_thread_inst_executed_op_fmul_pred_on.sum.per_cycle_elapsed",
    "smsp__sass_thread_inst_executed_op_fadd_pred_on.sum.per_cycle_elapsed",
]
STALLS = "smsp__average_warps_issue_stalled_"


def launches(path, out):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    agg = defaultdict(list)
    for r in rows[hi + 1:]:
        if len(r) > vi:
            agg[r[ki]].append(float(r[vi].replace(",", "")))
    tot = sum(sum(v) for v in agg.values())
    own = sum(sum(v) for k, v in agg.items() if "sbs" in k)
    with open(out, "w") as f:
        f.write(f"# ncu launch list ({path.split('/')[-1]}): gpu__time_duration.sum, cold-cache, serialised\n\n")
        f.write("| kernel | launches | avg us | share of all | share of sbs kernels |\n|---|---|---|---|---|\n")
        for k, v in sorted(agg.items(), key=lambda x: -sum(x[1])):
            f.write(f"| `{k[:70]}` | {len(v)} | {sum(v)/len(v)/1e3:.2f} | {sum(v)/tot:.3f} | "
                    f"{(sum(v)/own if 'sbs' in k else 0):.3f} |\n")
    print(open(out).read())


def full(rep, out, K, H):
    raw = subprocess.check_output(["ncu", "-i", rep, "--page", "raw", "--csv"]).decode()
    rows = list(csv.reader(io.StringIO(raw)))
    h, u = rows[0], rows[1]
    with open(out, "w") as f:
        for row in rows[2:]:
            name = row[h.index("Kernel Name")]
            f.write(f"# ncu --set full: `{name}` ({rep.split('/')[-1]}), K = {K}, H = {H}\n\n| metric | value | unit |\n|---|---|---|\n")
            g = {}
            for k in KEYS:
                if k in h:
                    f.write(f"| {k} | {row[h.index(k)]} | {u[h.index(k)]} |\n")
                    try:
                        g[k] = float(row[h.index(k)].replace(",", ""))
                    except ValueError:
                        pass
            t = g["gpu__time_duration.sum"] * (1e-3 if u[h.index("gpu__time_duration.sum")] == "ms" else 1e-6)
            cyc = t * g["sm__cycles_elapsed.avg.per_second"] * (1e9 if u[h.index("sm__cycles_elapsed.avg.per_second")] == "Ghz" else 1e6)
            rate = (2 * g[KEYS[-3]] + g[KEYS[-2]] + g[KEYS[-1]])
            flop = rate * cyc
            scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
            dram = sum(g[k] * scale.get(u[h.index(k)], 1.0) for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
            alg = 886.1419270833334 * K * H  # bench.py ALG_FLOP_FUSED (oracle op-counting mode) x units
            f.write(f"\nDerived: algorithmic FLOPs (oracle op count, 886.14 per sample-step) per launch = {alg:.4e}, "
                    f"{alg / t / 1e12:.2f} TFLOP/s under ncu ({alg / t / 74.45e12:.3f} of 74.45 TFLOP/s; ncu's clock "
                    f"{cyc / t / 1e6:.0f} MHz); instructions per sample = {g['inst_executed']*32/K:.0f}; "
                    f"scalar FFMA/FMUL/FADD counters alone (packed FFMA2/FADD2/FMUL2 not counted) = {flop/(K*H):.1f} "
                    f"FLOP per sample-step; DRAM bytes per launch = {dram:.4g}\n\n")
            st = sorted(((k[len(STALLS):].replace('_per_issue_active.ratio', ''), float(row[i] or 0))
                         for i, k in enumerate(h) if k.startswith(STALLS) and k.endswith("per_issue_active.ratio")),
                        key=lambda x: -x[1])
            f.write("Stall reasons (warps per issue-active cycle): " + ", ".join(f"{k} {v:.3f}" for k, v in st[:9]) + "\n\n")
    print(open(out).read())


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2], sys.argv[3])
    else:
        full(sys.argv[2], sys.argv[3], int(sys.argv[4]), int(sys.argv[5]))
