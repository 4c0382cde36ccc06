timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu_all.log 2>&1; echo pytest-all rc=$?; tail -3 gpurun_out/pytest_gpu_all.log
grep -E "^E " gpurun_out/pytest_gpu_all.log | head
echo "--- split"; timeout 300 python scripts/quick_time.py 2>&1 | grep -E "config|2\^1[68]"
echo "--- no split"; SBS_SPLIT=0 timeout 300 python scripts/quick_time.py 2>&1 | grep -E "config|2\^1[68]"
