# experiments: A/B latency of the in-tree build against libsbs_base.so (a build of an earlier commit)
for i in 1 2 3; do
SBS_LIB_PATH=$PWD/paper_2403_11383_b200/libsbs_base.so timeout 300 python scripts/ab_latency.py base
timeout 300 python scripts/ab_latency.py new
done
