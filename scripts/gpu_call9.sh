timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?; tail -5 gpurun_out/pytest_gpu.log
timeout 300 python scripts/quick_time.py > gpurun_out/qt.log 2>&1; echo qt rc=$?; cat gpurun_out/qt.log
python scripts/profile_step.py --workload c4 --steps 3 > gpurun_out/plain_c4.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:sbs_rollout -s 1 -c 1 -o gpurun_out/prof_c4_v2 python scripts/profile_step.py --workload c4 --steps 3 > gpurun_out/ncu_c4.log 2>&1; echo ncu rc=$?
