# full round check: GPU tests, smoke, bench (default flags), then the ncu launch list + one full capture of the fine kernel
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x --timeout 300 > gpurun_out/pytest_full.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_full.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench_full.log 2>&1
echo "bench rc=$?" >> gpurun_out/bench_full.log
if [ "${PROF:-1}" = "1" ]; then
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_bench.csv python bench.py --steps 1 --warmup 1 --no-parareal --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
  timeout 300 python scripts/prof_target.py fine > gpurun_out/plain_fine.log 2>&1 && \
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:rk3_march -s 1 -c 1 -o gpurun_out/fine_march python scripts/prof_target.py fine > gpurun_out/ncu_fine.log 2>&1
fi
