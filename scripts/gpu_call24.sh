timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/pytest_gpu.log
timeout 300 python scripts/quick_time.py 2>&1 | grep -E "config|2\^"
timeout 600 python bench.py --steps 3000 > gpurun_out/bench.log 2>&1; echo bench rc=$?; python -c "
import json; d=json.loads([l for l in open('gpurun_out/bench.log') if l.startswith('{')][-1]); print(d['value'], d['latency_us'], d['e2e'], d['roofline']['kernel_us'])"
