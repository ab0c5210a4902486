cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python scripts/prof_target.py coarse > gpurun_out/plain_coarse.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:fefb_tb -c 1 -o gpurun_out/coarse_v8 python scripts/prof_target.py coarse > gpurun_out/ncu_coarse8.log 2>&1
echo "rc=$?" >> gpurun_out/ncu_coarse8.log
