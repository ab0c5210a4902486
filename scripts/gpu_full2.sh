# round check: full GPU suite, smoke, default bench, launch list of the bench, ncu of K1
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
T=${TAG:-f2}
timeout 1500 python -m pytest tests -m gpu -q --timeout 600 > gpurun_out/pytest_$T.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_$T.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$T.log 2>&1
echo "smoke rc=$?" >> gpurun_out/smoke_$T.log
timeout 900 python bench.py > gpurun_out/bench_$T.log 2>&1
echo "bench rc=$?" >> gpurun_out/bench_$T.log
if [ "${PROF:-1}" = "1" ]; then
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_bench_$T.csv python bench.py --steps 1 --warmup 1 --no-parareal --no-cpu-baseline > gpurun_out/ncu_launch_$T.log 2>&1
  python scripts/launch_summary.py gpurun_out/launches_bench_$T.csv 20 > gpurun_out/launches_bench_$T.txt 2>&1
fi
