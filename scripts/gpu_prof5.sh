# launch list of one c3 window (cold single window; ncu serialises launches, compare shares only)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python scripts/prof_target.py c3k5 > gpurun_out/plain_c3k5.log 2>&1 && \
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c3k5_v6.csv python scripts/prof_target.py c3k5 > gpurun_out/ncu_c3k5.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_c3k5.log
