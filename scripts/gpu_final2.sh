# round-2 closing run: full GPU suite, smoke, default bench, reference arm, torchrun N=1 contract,
# launch list of the bench, ncu of K1 (200-step launch)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
T=${TAG:-fin2}
timeout 2400 python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/pytest_$T.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_$T.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$T.log 2>&1
echo "smoke rc=$?" >> gpurun_out/smoke_$T.log
timeout 900 python bench.py > gpurun_out/bench_$T.log 2>&1
echo "bench rc=$?" >> gpurun_out/bench_$T.log
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_$T.log 2>&1
echo "bench ref rc=$?" >> gpurun_out/bench_ref_$T.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 1 --steps 3 --warmup 3 --no-cpu-baseline --no-c4 > gpurun_out/torchrun1_$T.log 2>&1
echo "rc=$?" >> gpurun_out/torchrun1_$T.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_bench_$T.csv python bench.py --steps 1 --warmup 1 --no-parareal --no-cpu-baseline > gpurun_out/ncu_launch_$T.log 2>&1
python scripts/launch_summary.py gpurun_out/launches_bench_$T.csv 20 > gpurun_out/launches_bench_$T.txt 2>&1
timeout 300 python scripts/prof_target.py fine200 > gpurun_out/plain_fine200_$T.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:rk3_mtma -c 1 -f -o gpurun_out/mtma_$T python scripts/prof_target.py fine200 > gpurun_out/ncu_mtma_$T.log 2>&1
python scripts/ncu_summary.py gpurun_out/mtma_$T.ncu-rep --source 20 > gpurun_out/ncu_mtma_${T}_summary.txt 2>&1
tail -3 gpurun_out/pytest_$T.log; tail -2 gpurun_out/smoke_$T.log; tail -1 gpurun_out/bench_$T.log
