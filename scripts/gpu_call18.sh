timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/pytest_gpu.log
timeout 300 python scripts/quick_time.py 2>&1 | grep -E "config|2\^"
python scripts/profile_step.py --workload c3cem --steps 8 > gpurun_out/plain_c3.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"sbs_select|sbs_elite" -s 10 -c 2 -o gpurun_out/prof_c3b python scripts/profile_step.py --workload c3cem --steps 8 > gpurun_out/ncu_c3.log 2>&1; echo ncu rc=$?
