cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for v in 0 1 2 3 4 5 6 7; do
  PW_FUSED_VARIANT=$v timeout 120 python scripts/microbench.py fine >> gpurun_out/tune1.log 2>&1
done
timeout 600 python -m pytest tests/test_gpu_kernels.py -q -x --timeout 300 > gpurun_out/pytest_k.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_k.log
