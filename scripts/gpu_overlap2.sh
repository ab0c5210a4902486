cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
L=gpurun_out/overlap2.log
: > $L
for cfg in "0 0" "5 1" "0 1"; do
  set -- $cfg
  echo "coarse variant $1 overlap $2" >> $L
  PW_COARSE_VARIANT=$1 PW_SWEEP_OVERLAP=$2 timeout 300 python scripts/c3_window.py >> $L 2>&1
done
PW_COARSE_VARIANT=5 PW_SWEEP_OVERLAP=1 timeout 600 python -m pytest tests/test_gpu_sweeps.py -m gpu -q -x --timeout 300 >> $L 2>&1
