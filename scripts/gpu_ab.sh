# quick fine-kernel check: march parity tests + c2 / c3-grid throughput (no profiler); extra env via AB_ENV
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
L=gpurun_out/ab.log
: > $L
timeout 300 python -m pytest tests/test_gpu_march.py -q -x -m gpu 2>&1 | tail -1 >> $L
for w in fine fine512; do
  timeout 120 python scripts/microbench.py $w 2>&1 | grep -E "10 step|4 steps" >> $L
done
if [ -n "$AB_ENV" ]; then
  echo "== $AB_ENV" >> $L
  env $AB_ENV timeout 300 python -m pytest tests/test_gpu_march.py -q -x -m gpu 2>&1 | tail -1 >> $L
  for w in fine fine512; do
    env $AB_ENV timeout 120 python scripts/microbench.py $w 2>&1 | grep -E "rel err|10 step|4 steps" >> $L
  done
fi
