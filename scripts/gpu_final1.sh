# floors printout, torchrun N=1 contract, ncu of the current K1 (fine200) and its launch list
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
T=${TAG:-fin}
timeout 900 python -m pytest tests/test_gpu_windows_ref.py tests/test_gpu_sweeps.py -q -s --timeout 600 > gpurun_out/floors_$T.log 2>&1
echo "rc=$?" >> gpurun_out/floors_$T.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 1 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/torchrun1_$T.log 2>&1
echo "rc=$?" >> gpurun_out/torchrun1_$T.log
timeout 300 python scripts/prof_target.py fine200 > gpurun_out/plain_fine200_$T.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:rk3_mtma -c 1 -o gpurun_out/mtma_$T python scripts/prof_target.py fine200 > gpurun_out/ncu_mtma_$T.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c3k5_$T.csv python scripts/prof_target.py c3k5 > /dev/null 2>&1
python scripts/launch_summary.py gpurun_out/launches_c3k5_$T.csv 40 > gpurun_out/launches_c3k5_$T.txt 2>&1
