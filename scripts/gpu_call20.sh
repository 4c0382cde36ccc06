python scripts/profile_step.py --workload c3cem --steps 8 > gpurun_out/plain_c3.log 2>&1 && \
ncu --set full --warp-sampling-interval 0 --clock-control none --import-source on -k regex:"sbs_cem" -s 5 -c 1 -o gpurun_out/prof_cem python scripts/profile_step.py --workload c3cem --steps 8 > gpurun_out/ncu_cem.log 2>&1; echo ncu rc=$?
