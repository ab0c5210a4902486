# row-marching fine kernel: parity tests, then throughput of each variant (no profiler)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
L=gpurun_out/march.log
: > $L
timeout 600 python -m pytest tests/test_gpu_march.py tests/test_gpu_kernels.py -m gpu -q -x --timeout 300 >> $L 2>&1
echo "pytest rc=$?" >> $L
for cfg in "PW_MARCH=0" "PW_MARCH=1" ${EXTRA_CFGS}; do
  echo "== $cfg" >> $L
  env $cfg timeout 120 python scripts/microbench.py fine >> $L 2>&1
done
