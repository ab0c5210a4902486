# env-variant sweep of the fine microbench (no profiler): CFGS="A=1 B=2|A=2" (| separates runs)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
L=gpurun_out/sweep.log
: > $L
IFS='|' read -ra RUNS <<< "$CFGS"
for cfg in "${RUNS[@]}"; do
  echo "== $cfg" >> $L
  env $cfg timeout 120 python scripts/microbench.py ${WHAT:-fine} 2>&1 | grep -E "10 step|4 steps" >> $L
done
