#!/bin/bash
# compute-sanitizer (memcheck, racecheck, synccheck) over small shapes of every kernel family
# (tools/sanitize_driver.py); logs -> gpurun_out/sanitize/ (summaries copied to profiles/).
cd ${GRAFT_REPO_ROOT:-.}
O=gpurun_out/sanitize; mkdir -p $O
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck synccheck racecheck; do
  for fam in mix dL trace normal shard d1d; do
    timeout 900 $CS --tool $tool --print-limit 50 --error-exitcode 9 \
      python tools/sanitize_driver.py $fam > $O/${tool}_${fam}.log 2>&1
    echo "$tool $fam rc=$?" >> $O/summary.txt
  done
done
cat $O/summary.txt
