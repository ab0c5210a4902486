# session baseline: full GPU suite, default bench, smoke
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
T=${TAG:-s5}
timeout 1500 python -m pytest tests -m gpu -x -q --timeout 900 > gpurun_out/pytest_$T.log 2>&1
echo "rc=$?" >> gpurun_out/pytest_$T.log
timeout 600 python bench.py > gpurun_out/bench_$T.log 2>&1
echo "rc=$?" >> gpurun_out/bench_$T.log
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke_$T.log 2>&1
echo "rc=$?" >> gpurun_out/smoke_$T.log
tail -3 gpurun_out/pytest_$T.log; tail -2 gpurun_out/bench_$T.log; tail -2 gpurun_out/smoke_$T.log
