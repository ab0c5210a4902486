# K1 with 8 columns per thread (PW_MARCH_BX=8): parity tests under the variant, then c2 bench A/B
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
T=${TAG:-bx8}
PW_MARCH_BX=8 timeout 900 python -m pytest tests/test_gpu_march.py tests/test_gpu_bench_config.py -q -x --timeout 300 > gpurun_out/pytest_$T.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_$T.log
: > gpurun_out/sweep_$T.log
for V in ${VARIANTS:-PW_MARCH_BX=4 PW_MARCH_BX=8 PW_MARCH_UNI=1}; do
  env $V timeout 300 python bench.py --no-parareal --no-cpu-baseline --steps 5 > gpurun_out/b.tmp 2>&1
  python -c "
import json,sys
for l in open('gpurun_out/b.tmp'):
    if l.startswith('{'):
        d=json.loads(l); print('$V', round(d['value']/1e9,2), 'G/s frac', round(d['roofline']['frac'],4), 'e2e', round(d['e2e']['value']/1e9,2))
" >> gpurun_out/sweep_$T.log 2>&1
  tail -3 gpurun_out/b.tmp | cut -c1-300 >> gpurun_out/sweep_$T.log
done
cat gpurun_out/sweep_$T.log; tail -5 gpurun_out/pytest_$T.log
