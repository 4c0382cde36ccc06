timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu_all.log 2>&1; echo pytest-all rc=$?; tail -2 gpurun_out/pytest_gpu_all.log
grep -E "^E " gpurun_out/pytest_gpu_all.log | head
python scripts/phase_times.py 2>&1 | tail -4
timeout 300 python scripts/quick_time.py 2>&1 | grep -E "config|2\^1[68]|2\^22"
