cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
T=${TAG:-tq}
timeout 600 python -m pytest tests/test_gpu_tsqr.py -q -x --timeout 300 > gpurun_out/pytest_$T.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_$T.log
timeout 300 python scripts/qr_bench.py > gpurun_out/qr_$T.log 2>&1
QR_REPS=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_qrc3_$T.csv python scripts/qr_bench.py 786432 64 > /dev/null 2>&1
python scripts/launch_summary.py gpurun_out/launches_qrc3_$T.csv 30 > gpurun_out/launches_qrc3_$T.txt 2>&1
