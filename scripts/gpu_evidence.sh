# round evidence in one gpurun call: bench line, reference arm, ncu launch list of a short
# bench run, ncu --set full of the K = 2^22 and config-2 rollouts and of the CEM kernels
set -x
python bench.py > gpurun_out/bench.log 2>&1; echo bench rc=$?; tail -1 gpurun_out/bench.log
python bench.py --impl reference --steps 20 --warmup 3 > gpurun_out/bench_ref.log 2>&1; echo ref rc=$?; tail -1 gpurun_out/bench_ref.log
python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-other-configs --e2e-steps 5 > gpurun_out/plain_small.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-other-configs --e2e-steps 5 > gpurun_out/ncu_launch.log 2>&1; echo ncu1 rc=$?
python scripts/profile_step.py --workload c4 --steps 3 > gpurun_out/plain_c4.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:sbs_rollout -s 1 -c 1 -f -o gpurun_out/prof_c4 python scripts/profile_step.py --workload c4 --steps 3 > gpurun_out/ncu_c4.log 2>&1; echo ncu2 rc=$?
python scripts/profile_step.py --workload c2 --steps 8 > gpurun_out/plain_c2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:sbs_rollout -s 5 -c 1 -f -o gpurun_out/prof_c2 python scripts/profile_step.py --workload c2 --steps 8 > gpurun_out/ncu_c2.log 2>&1; echo ncu3 rc=$?
python scripts/profile_step.py --workload c3cem --steps 8 > gpurun_out/plain_c3.log 2>&1 && \
ncu --set full --clock-control none -k regex:"sbs_" -s 12 -c 3 -f -o gpurun_out/prof_c3 python scripts/profile_step.py --workload c3cem --steps 8 > gpurun_out/ncu_c3.log 2>&1; echo ncu4 rc=$?
