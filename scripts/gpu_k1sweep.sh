# K1 variants: parity tests, then c2 bench under env variants (one line each)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
T=${TAG:-k1s}
timeout 600 python -m pytest tests/test_gpu_march.py tests/test_gpu_bench_config.py -q -x --timeout 300 > gpurun_out/pytest_$T.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_$T.log
: > gpurun_out/sweep_$T.log
for V in ${VARIANTS:-"X=0"}; do
  env $V timeout 300 python bench.py --no-parareal --no-cpu-baseline --steps 5 > gpurun_out/b.tmp 2>&1
  python -c "
import json,sys
for l in open('gpurun_out/b.tmp'):
    if l.startswith('{'):
        d=json.loads(l); print('$V', round(d['value']/1e9,2), 'G/s frac', round(d['roofline']['frac'],4), 'e2e', round(d['e2e']['value']/1e9,2))
" >> gpurun_out/sweep_$T.log 2>&1
done
