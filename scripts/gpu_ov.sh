# overlapped serial correction: parity with PW_SERIAL_OVERLAP=1, window times off / on
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
T=${TAG:-ov}
PW_SERIAL_OVERLAP=1 timeout 1200 python -m pytest tests/test_gpu_sweeps.py tests/test_gpu_windows_ref.py -q -x --timeout 600 > gpurun_out/pytest_$T.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_$T.log
for V in 0 1; do
  PW_SERIAL_OVERLAP=$V timeout 900 python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/b.tmp 2>&1
  python -c "
import json
for l in open('gpurun_out/b.tmp'):
    if l.startswith('{'):
        d=json.loads(l); p=d['parareal']; p4=d.get('parareal_c4',{})
        print('OVERLAP=$V c3', round(p['window_s'],4), {k: round(v,4) for k,v in p['phases_s'].items()}, p['ranks'])
        print('OVERLAP=$V c4', p4.get('window_s'), p4.get('phases_s'), p4.get('ranks'))
" >> gpurun_out/ov_$T.log 2>&1
done
