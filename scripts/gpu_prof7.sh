# launch list of the subspace-refactorisation kernels of one c4 window (serial-step, coarse and
# fine kernels excluded from the capture)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python scripts/prof_target.py c4k4 > gpurun_out/plain_c4k4.log 2>&1 && \
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -k 'regex:^(?!.*(combine|fefb|rk3|reduce_parts|residual|axpby|colmax|sqdiff)).*' --csv --log-file gpurun_out/launches_c4qr.csv python scripts/prof_target.py c4k4 > gpurun_out/ncu_c4qr.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_c4qr.log
