timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/pytest_gpu.log
for v in "" _mb3; do echo "== lib$v"; SBS_LIB_PATH=$PWD/paper_2403_11383_b200/libsbs$v.so timeout 300 python scripts/quick_time.py 2>&1 | grep -E "config|2\^" ; done
