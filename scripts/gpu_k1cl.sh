cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
T=${TAG:-cl}
timeout 900 python -m pytest tests/test_gpu_march.py -q -x --timeout 300 -k "cluster or grids" > gpurun_out/pytest_$T.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_$T.log
timeout 300 python scripts/microbench.py wide > gpurun_out/fine_$T.log 2>&1
PW_MARCH_CLUSTER2=0 timeout 300 python scripts/microbench.py wide >> gpurun_out/fine_$T.log 2>&1
