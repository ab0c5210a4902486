# ncu --set full of the serial-step kernels inside a c3 window (K=2): the TMA GEMV and the
# temporal-blocked coarse G (each capture after the plain run exited 0)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python scripts/prof_target.py c3k2 > gpurun_out/plain_c3k2.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:combine_tma -s 100 -c 1 -o gpurun_out/gemv_tma_v1 python scripts/prof_target.py c3k2 > gpurun_out/ncu_gemv.log 2>&1
echo "ncu1 rc=$?" >> gpurun_out/ncu_gemv.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fefb_tb -s 20 -c 1 -o gpurun_out/coarse_v7 python scripts/prof_target.py c3k2 > gpurun_out/ncu_coarse7.log 2>&1
echo "ncu2 rc=$?" >> gpurun_out/ncu_coarse7.log
