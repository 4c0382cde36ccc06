timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?; tail -5 gpurun_out/pytest_gpu.log
timeout 300 python scripts/quick_time.py > gpurun_out/qt.log 2>&1; echo qt rc=$?; cat gpurun_out/qt.log
python scripts/profile_step.py --workload c3cem > gpurun_out/plain_c3.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"sbs_select|sbs_elite|sbs_rollout" -s 6 -c 3 -o gpurun_out/prof_c3cem python scripts/profile_step.py --workload c3cem > gpurun_out/ncu_c3.log 2>&1; echo ncu rc=$?
