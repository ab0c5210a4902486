cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
T=${TAG:-nf}
timeout 900 python -m pytest tests/test_gpu_coarse_nf.py -q -x --timeout 300 > gpurun_out/pytest_$T.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_$T.log
: > gpurun_out/coarse_$T.log
for V in 0 2 3 4; do echo "PW_COARSE_NF=$V" >> gpurun_out/coarse_$T.log; PW_COARSE_NF=$V timeout 120 python scripts/microbench.py coarse >> gpurun_out/coarse_$T.log 2>&1; done
