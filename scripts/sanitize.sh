# compute-sanitizer over the library's kernels: one tool per call,
#   bash scripts/sanitize.sh memcheck|racecheck|synccheck|initcheck
# every command below also runs clean without the tool (scripts/profile_step.py, pytest).
tool=${1:-memcheck}
out=gpurun_out/sanitize_${tool}.log
CS="compute-sanitizer --tool ${tool} --kernel-name kns=sbs_ --error-exitcode 7 --print-limit 50"
[ "$tool" = "racecheck" ] && CS="$CS --racecheck-report all"
: > $out
run() { echo "=== $*" >> $out; timeout 1200 $CS "$@" >> $out 2>&1; echo "=== rc=$?" >> $out; }
run python scripts/profile_step.py --workload c1 --steps 2             # latency mode, producer/integrator warps, MPPI
run python scripts/profile_step.py --workload c3cem --steps 2          # CEM: rollout + select + elite under PDL
run python scripts/profile_step.py --workload c3naive --steps 2        # Naive: fused argmin tail
run python scripts/profile_step.py --workload c4 --K 65536 --steps 2   # throughput mode, chunked MPPI merge
run python -m pytest tests/test_gpu_parity.py -q -x -k "peer_memory_exchange and mppi-10000-2-1-1" # peer-memory exchange, 2 contexts
run python -m pytest tests/test_gpu_loop.py -q -x -k "run_loop_equals_stepwise"  # closed loop (advance kernel, graphs)
run python -m pytest tests/test_gpu_fullcov.py -q -x -k "iterations_match_oracle"        # full-covariance CEM (cov kernel)
grep -E "^=== |ERROR SUMMARY|RACECHECK SUMMARY|Invalid|Race|Hazard|error" $out | head -80
