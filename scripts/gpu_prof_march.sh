# ncu --set full of the row-marching fine kernel (after a plain run exits 0); env passes through
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
V=${V:-march_v1}
timeout 300 python scripts/prof_target.py fine > gpurun_out/plain_$V.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:rk3_march -s 1 -c 1 -o gpurun_out/$V python scripts/prof_target.py fine > gpurun_out/ncu_$V.log 2>&1
echo "rc=$?" >> gpurun_out/ncu_$V.log
