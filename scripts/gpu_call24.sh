timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu_all.log 2>&1; echo pytest-all rc=$?; tail -3 gpurun_out/pytest_gpu_all.log
grep -E "^E " gpurun_out/pytest_gpu_all.log | head
timeout 600 python bench.py > gpurun_out/bench.jsonl 2> gpurun_out/bench.err; echo bench rc=$?; tail -3 gpurun_out/bench.err
