# panel QR launch breakdown (c3 / c4 shapes) + K1 bench
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
T=${TAG:-qp}
timeout 300 python scripts/qr_bench.py 786432 64 > gpurun_out/qr_c3_$T.log 2>&1
timeout 300 python scripts/qr_bench.py 3145728 256 > gpurun_out/qr_c4_$T.log 2>&1
QR_REPS=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_qrc3_$T.csv python scripts/qr_bench.py 786432 64 > /dev/null 2>&1
python scripts/launch_summary.py gpurun_out/launches_qrc3_$T.csv 30 > gpurun_out/launches_qrc3_$T.txt 2>&1
QR_REPS=1 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_qrc4_$T.csv python scripts/qr_bench.py 3145728 256 > /dev/null 2>&1
python scripts/launch_summary.py gpurun_out/launches_qrc4_$T.csv 30 > gpurun_out/launches_qrc4_$T.txt 2>&1
timeout 300 python bench.py --no-parareal --no-cpu-baseline > gpurun_out/bench_$T.log 2>&1
