cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python scripts/microbench.py ${1:-coarse} > gpurun_out/quick.log 2>&1
timeout 600 python -m pytest tests -m gpu -q -x --timeout 300 > gpurun_out/pytest_quick.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_quick.log
