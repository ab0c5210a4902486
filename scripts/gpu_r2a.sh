# round-2 checkpoint: GPU suite, smoke, QR microbench, default bench
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q --timeout 400 > gpurun_out/pytest_r2a.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_r2a.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r2a.log 2>&1
echo "smoke rc=$?" >> gpurun_out/smoke_r2a.log
timeout 300 python scripts/qr_bench.py > gpurun_out/qr_r2a.log 2>&1
echo "qr rc=$?" >> gpurun_out/qr_r2a.log
timeout 900 python bench.py > gpurun_out/bench_r2a.log 2>&1
echo "bench rc=$?" >> gpurun_out/bench_r2a.log
