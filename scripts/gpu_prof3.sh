cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python scripts/prof_target.py c3k5 > gpurun_out/plain_c3k5.log 2>&1 && \
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c3k5.csv python scripts/prof_target.py c3k5 > gpurun_out/ncu_c3k5.log 2>&1
echo "ncu1 rc=$?" >> gpurun_out/ncu_c3k5.log
timeout 300 python scripts/prof_target.py coarse > gpurun_out/plain_coarse.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:fefb_coop -c 1 -o gpurun_out/coarse_v2 python scripts/prof_target.py coarse > gpurun_out/ncu_coarse.log 2>&1
echo "ncu2 rc=$?" >> gpurun_out/ncu_coarse.log
