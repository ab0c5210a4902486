cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
(timeout 300 python scripts/microbench.py coarse; PW_QR_TIMING=1 timeout 300 python scripts/prof_target.py c3k2) > gpurun_out/coarse.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -x --timeout 300 > gpurun_out/pytest_all.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_all.log
timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_q.log 2>&1
