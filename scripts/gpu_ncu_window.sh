# ncu --set full of one launch each of the window's other kernels (coarse G, serial combine pass,
# TSQR leaf, DMMA GEMM) inside a c3 K=2 window; summaries by scripts/ncu_summary.py
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
T=${TAG:-win}
timeout 300 python scripts/prof_target.py c3k2 > gpurun_out/plain_c3k2_$T.log 2>&1 || exit 1
for spec in "fefb_nfr:100:coarse_g" "combine_tma:100:combine" "tsqr_qr_kernel:2:tsqr_leaf" "dgemm_kernel:6:dgemm"; do
  K=${spec%%:*}; rest=${spec#*:}; SKIP=${rest%%:*}; NAME=${rest#*:}
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$K --launch-skip $SKIP -c 1 -f \
    -o gpurun_out/${NAME}_$T python scripts/prof_target.py c3k2 > gpurun_out/ncu_${NAME}_$T.log 2>&1
  python scripts/ncu_summary.py gpurun_out/${NAME}_$T.ncu-rep --source 12 > gpurun_out/ncu_${NAME}_${T}_summary.txt 2>&1
  echo "== $NAME"; head -30 gpurun_out/ncu_${NAME}_${T}_summary.txt | grep "Duration\|DRAM Throughput\|Issue Slots\|Registers\|Achieved Occ\|L1/TEX Cache\|Compute (SM)"; tail -2 gpurun_out/ncu_${NAME}_${T}_summary.txt
done
