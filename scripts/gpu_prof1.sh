cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python scripts/microbench.py all > gpurun_out/micro.log 2>&1
echo "micro rc=$?" >> gpurun_out/micro.log
timeout 300 python scripts/prof_target.py c3k2 > gpurun_out/plain_c3k2.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c3k2.csv python scripts/prof_target.py c3k2 > gpurun_out/ncu_c3k2.log 2>&1
echo "ncu1 rc=$?" >> gpurun_out/ncu_c3k2.log
timeout 300 python scripts/prof_target.py fine > gpurun_out/plain_fine.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:rk3_fused -s 1 -c 1 -o gpurun_out/fine_v1 python scripts/prof_target.py fine > gpurun_out/ncu_fine.log 2>&1
echo "ncu2 rc=$?" >> gpurun_out/ncu_fine.log
