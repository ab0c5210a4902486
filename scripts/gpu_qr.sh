cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q -x --timeout 300 > gpurun_out/pytest_quick.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_quick.log
PW_WARM=1 PW_QR_TIMING=1 timeout 300 python scripts/prof_target.py c3k5 > gpurun_out/qrt.log 2>&1
