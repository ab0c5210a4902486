# K1 check: march parity tests, c2 bench (new vs previous kernel), optional ncu of the persistent launch
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
T=${TAG:-k1}
timeout 600 python -m pytest tests/test_gpu_march.py tests/test_gpu_bench_config.py -q -x --timeout 300 > gpurun_out/pytest_$T.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_$T.log
timeout 300 python bench.py --no-parareal --no-cpu-baseline > gpurun_out/bench_$T.log 2>&1
echo "bench rc=$?" >> gpurun_out/bench_$T.log
PW_MARCH_V2=0 timeout 300 python bench.py --no-parareal --no-cpu-baseline > gpurun_out/bench_${T}_old.log 2>&1
if [ "${PROF:-0}" = "1" ]; then
  timeout 300 python scripts/prof_target.py fine200 > gpurun_out/plain_fine200_$T.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:rk3_mtma -c 1 -o gpurun_out/mtma_$T python scripts/prof_target.py fine200 > gpurun_out/ncu_mtma_$T.log 2>&1
fi
