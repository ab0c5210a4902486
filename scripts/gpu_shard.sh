cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
L=gpurun_out/shard.log
timeout 900 python -m pytest tests -m gpu -q -x --timeout 300 > $L 2>&1
echo "pytest rc=$?" >> $L
for n in 1 4; do
  echo "row shards $n" >> $L
  PW_ROW_SHARDS=$n timeout 300 python scripts/c3_window.py >> $L 2>&1
done
