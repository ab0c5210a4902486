# G with phase A folded into the first substep block (PW_COARSE_NF=6) vs the phase-A form (3)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
T=${TAG:-nf4}
timeout 900 python -m pytest tests/test_gpu_coarse_nf.py -q -x --timeout 300 > gpurun_out/pytest_$T.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_$T.log
: > gpurun_out/coarse_$T.log
for V in ${VARIANTS:-3 6}; do echo "PW_COARSE_NF=$V" >> gpurun_out/coarse_$T.log; PW_COARSE_NF=$V timeout 120 python scripts/microbench.py coarse >> gpurun_out/coarse_$T.log 2>&1; done
for V in ${BENCHV:-3 6}; do
  PW_COARSE_NF=$V timeout 900 python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/b.tmp 2>&1
  python -c "
import json
for l in open('gpurun_out/b.tmp'):
    if l.startswith('{'):
        d=json.loads(l); p=d['parareal']; p4=d.get('parareal_c4',{})
        print('NF=$V c3', round(p['window_s'],4), {k: round(v,4) for k,v in p['phases_s'].items()})
        print('NF=$V c4', p4.get('window_s'), p4.get('phases_s'))
" >> gpurun_out/coarse_$T.log 2>&1
done
