#!/bin/bash
# fused gradient+mix A/B over the step kinds: RAD sync / stale, D1D (uniform, stale), fp64
cd "${GRAFT_REPO_ROOT:-/root/repo}"
o=gpurun_out/${1:-fused11}
mkdir -p $o
timeout 900 python -m pytest tests/test_gpu_fused_grad.py -x -q 2>&1 | tail -3 > $o/tests.log
for args in "64 25557032 7 0 0" "64 25557032 7 1 0" "64 25557032 7 1 1" "64 25557032 7 0 1" "16 1048576 20 1 0" "16 1048576 20 0 0"; do
  timeout 600 python tools/bench_fused_grad.py $args >> $o/ab.json 2>> $o/ab.err
done
cat $o/tests.log $o/ab.json
