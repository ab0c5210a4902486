# fine-kernel iteration: variant check vs oracle + throughput, then the fine GPU tests
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
L=gpurun_out/fine.log
: > $L
for v in ${VARIANTS:-0}; do
  PW_FUSED_VARIANT=$v timeout 120 python scripts/microbench.py fine >> $L 2>&1
done
timeout 600 python -m pytest tests/test_gpu_kernels.py -m gpu -q -x --timeout 300 >> $L 2>&1
echo "pytest rc=$?" >> $L
