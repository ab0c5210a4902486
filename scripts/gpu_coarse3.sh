cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
L=gpurun_out/coarse3.log
: > $L
for v in ${VARIANTS:-0 3}; do
  echo "variant $v" >> $L
  PW_COARSE_VARIANT=$v timeout 120 python scripts/microbench.py coarse >> $L 2>&1
  PW_COARSE_VARIANT=$v timeout 300 python -m pytest tests/test_gpu_kernels.py -m gpu -q -x -k "coarse or fefb or strict" --timeout 200 >> $L 2>&1
  PW_COARSE_VARIANT=$v timeout 300 python scripts/c3_window.py >> $L 2>&1
done
