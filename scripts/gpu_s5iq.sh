# implicit-Q A/B: window parity tests, then c3 / c4 window timings with and without
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
T=${TAG:-iq}
timeout 1500 python -m pytest tests/test_gpu_windows_ref.py tests/test_gpu_sweeps.py tests/test_gpu_runner.py tests/test_gpu_configs.py -x -q -s --timeout 900 > gpurun_out/pytest_$T.log 2>&1
echo "rc=$?" >> gpurun_out/pytest_$T.log
tail -3 gpurun_out/pytest_$T.log
for IQ in 1 0; do
  PW_IMPLICIT_Q=$IQ timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/bench_${T}_iq$IQ.log 2>&1
  echo "rc=$?" >> gpurun_out/bench_${T}_iq$IQ.log
  python - <<P
import json
for l in open("gpurun_out/bench_${T}_iq$IQ.log"):
    if l.startswith("{"):
        d=json.loads(l)
        for k in ("parareal","parareal_c4"):
            w=d.get(k,{})
            print("IQ=$IQ",k,w.get("window_s"),w.get("phases_s"),w.get("ranks"))
        print(d["roofline"].get("shared"))
P
done
