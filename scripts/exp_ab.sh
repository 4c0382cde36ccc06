set -x
for i in 1 2; do
AB_BIG=1 SBS_LIB_PATH=$PWD/paper_2403_11383_b200/libsbs_base.so timeout 300 python scripts/ab_latency.py base
AB_BIG=1 timeout 300 python scripts/ab_latency.py model
AB_BIG=1 SBS_MODEL=0 timeout 300 python scripts/ab_latency.py generic
done
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
