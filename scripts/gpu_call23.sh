timeout 900 python -m pytest tests/test_gpu_fullcov.py -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/pytest_gpu.log
grep -E "^E |Error" gpurun_out/pytest_gpu.log | head -20
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu_all.log 2>&1; echo pytest-all rc=$?; tail -3 gpurun_out/pytest_gpu_all.log
