timeout 900 python -m pytest tests/test_gpu_loop.py tests/test_gpu_closed_loop_trends.py -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?; tail -5 gpurun_out/pytest_gpu.log
grep -E "^E " gpurun_out/pytest_gpu.log | head -20
