# experiments: A/B of variant libraries (scripts/exp_build.py) -- device latency per iteration
for i in 1 2; do
for v in "$@"; do
AB_BIG=1 SBS_LIB_PATH=$PWD/paper_2403_11383_b200/libsbs_$v.so timeout 300 python scripts/ab_latency.py $v
done
done
