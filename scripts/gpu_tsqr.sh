cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
T=${TAG:-ts}
timeout 1200 python -m pytest tests/test_gpu_tsqr.py tests/test_gpu_dgemm.py tests/test_gpu_windows_ref.py tests/test_gpu_sweeps.py -q -x --timeout 600 > gpurun_out/pytest_$T.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_$T.log
timeout 300 python scripts/qr_bench.py > gpurun_out/qr_$T.log 2>&1
QR_REPS=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_qrc3_$T.csv python scripts/qr_bench.py 786432 64 > /dev/null 2>&1
python scripts/launch_summary.py gpurun_out/launches_qrc3_$T.csv 30 > gpurun_out/launches_qrc3_$T.txt 2>&1
PW_WARM=1 PW_QR_TIMING=1 timeout 300 python scripts/prof_target.py c3k5 > gpurun_out/qrt_c3_$T.log 2>&1
