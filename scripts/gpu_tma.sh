cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
L=gpurun_out/tma.log
: > $L
for v in 0 5; do
  echo "variant $v" >> $L
  PW_CG_VARIANT=$v timeout 60 ./scripts/ubench_gemv >> $L 2>&1
  PW_CG_VARIANT=$v timeout 300 python scripts/c3_window.py >> $L 2>&1
done
PW_CG_VARIANT=5 timeout 600 python -m pytest tests/test_gpu_sweeps.py tests/test_gpu_windows_ref.py -m gpu -q -x --timeout 300 >> $L 2>&1
