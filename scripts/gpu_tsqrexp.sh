# TSQR leaf experiment: libraries differing only in the leaf kernel (original; xj re-read after
# the barrier with __launch_bounds__ min blocks 1 / 4 / 5)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
L=paper_1510_02237_b200/libpitwave_b200.so
cp $L /tmp/lib_default.so
: > gpurun_out/tsqrexp.log
for f in build/tsqrexp/lib_*.so; do
  cp $f $L
  echo "== $(basename $f)" >> gpurun_out/tsqrexp.log
  timeout 300 python -m pytest tests/test_gpu_tsqr.py -q -x --timeout 300 2>&1 | tail -1 >> gpurun_out/tsqrexp.log
  timeout 300 python scripts/qr_bench.py >> gpurun_out/tsqrexp.log 2>&1
done
cp /tmp/lib_default.so $L
