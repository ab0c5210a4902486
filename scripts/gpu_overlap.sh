cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
L=gpurun_out/overlap.log
: > $L
for cfg in "1 0" "1 1" "0 0"; do
  set -- $cfg
  PW_SWEEP_OVERLAP=$1 PW_COOP_CAP=$2 timeout 300 python scripts/c3_window.py >> $L 2>&1
done
timeout 900 python -m pytest tests -m gpu -q -x --timeout 300 > gpurun_out/pytest_quick.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_quick.log
