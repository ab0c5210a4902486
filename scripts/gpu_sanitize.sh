# compute-sanitizer over the reduced-shape protocol cases (scripts/sanitize_target.py)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/sanitize
CS=/usr/local/cuda/bin/compute-sanitizer
for case in march window peers; do
  timeout 600 python scripts/sanitize_target.py $case > gpurun_out/sanitize/plain_$case.log 2>&1 || echo "plain $case failed" >> gpurun_out/sanitize/plain_$case.log
  for tool in memcheck racecheck synccheck; do
    extra=""
    [ $tool = memcheck ] && extra="--leak-check no"
    timeout 1200 $CS --tool $tool $extra --print-limit 50 python scripts/sanitize_target.py $case \
      > gpurun_out/sanitize/${tool}_$case.log 2>&1
    echo "exit=$?" >> gpurun_out/sanitize/${tool}_$case.log
  done
done
grep -H "ERROR SUMMARY\|exit=\|ok" gpurun_out/sanitize/*.log
