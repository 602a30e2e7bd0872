#!/bin/bash
set -x
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out/fused7
timeout 900 python -m pytest tests/test_gpu_fused_grad.py -x -q 2>&1 | tail -5 > gpurun_out/fused7/tests.log
timeout 600 python tools/bench_fused_grad.py > gpurun_out/fused7/c2.json 2> gpurun_out/fused7/c2.err
timeout 600 python tools/bench_fused_grad.py 64 25557032 7 1 > gpurun_out/fused7/c2_stale.json 2>> gpurun_out/fused7/c2.err
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  -k regex:mix_tma --log-file gpurun_out/fused7/launches.csv python tools/bench_fused_grad.py 64 25557032 1 > gpurun_out/fused7/ncu.log 2>&1
cat gpurun_out/fused7/tests.log gpurun_out/fused7/c2.json gpurun_out/fused7/c2_stale.json
