cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
T=${TAG:-sp}
timeout 900 python -m pytest tests/test_gpu_march.py tests/test_gpu_bench_config.py tests/test_gpu_peer_gather.py -q -x --timeout 300 > gpurun_out/pytest_$T.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_$T.log
timeout 300 python bench.py --no-parareal --no-cpu-baseline > gpurun_out/bench_$T.log 2>&1
timeout 300 python scripts/microbench.py wide > gpurun_out/fine_$T.log 2>&1
