# ncu --set full of the 200-step K1 launch under an env variant (VAR="PW_MARCH_BX=8"), summary next to it
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
T=${TAG:-k1v}
env $VAR timeout 300 python scripts/prof_target.py fine200 > gpurun_out/plain_fine200_$T.log 2>&1 && \
env $VAR timeout 900 ncu --set full --clock-control none --import-source on -k regex:rk3_mtma -c 1 -f -o gpurun_out/mtma_$T python scripts/prof_target.py fine200 > gpurun_out/ncu_mtma_$T.log 2>&1
python scripts/ncu_summary.py gpurun_out/mtma_$T.ncu-rep --source 25 > gpurun_out/ncu_mtma_${T}_summary.txt 2>&1
head -60 gpurun_out/ncu_mtma_${T}_summary.txt
