# QR breakdown: per-phase CUDA-event marks of the refactorisation (c3 K=5, c4 K=4), GEMM bench, c3 launch list
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
PW_WARM=1 PW_QR_TIMING=1 timeout 300 python scripts/prof_target.py c3k5 > gpurun_out/qrt_c3.log 2>&1
PW_QR_TIMING=1 timeout 300 python scripts/prof_target.py c4k4 > gpurun_out/qrt_c4.log 2>&1
timeout 300 python scripts/gemm_bench.py > gpurun_out/gemm_r2b.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c3k5.csv python scripts/prof_target.py c3k5 > gpurun_out/ncu_c3k5.log 2>&1
python scripts/launch_summary.py gpurun_out/launches_c3k5.csv 40 > gpurun_out/launches_c3k5.txt 2>&1
