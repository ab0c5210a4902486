cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python scripts/prof_target.py fine > gpurun_out/plain_fine2.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:rk3_fused -s 1 -c 1 -o gpurun_out/fine_v5 python scripts/prof_target.py fine > gpurun_out/ncu_fine2.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_fine2.log
