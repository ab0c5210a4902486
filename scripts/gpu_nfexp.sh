# G flag-protocol experiment: nanosleep in the neighbour poll (s) and the explicit fence before
# the release store (f), each library built with -DNF_SLEEP / -DNF_FENCE
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
L=paper_1510_02237_b200/libpitwave_b200.so
cp $L /tmp/lib_default.so
: > gpurun_out/nfexp.log
for f in build/nfexp/lib_s*_f*.so; do
  cp $f $L
  for V in 11 12; do echo "$(basename $f) V=$V" >> gpurun_out/nfexp.log; PW_COARSE_NF=$V timeout 120 python scripts/microbench.py coarse 2>&1 | grep "FE-FB" >> gpurun_out/nfexp.log; done
done
cp /tmp/lib_default.so $L
