#!/bin/bash
# fused gradient + mix: parity tests, C2 timing, launch list
set -x
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out/fused
timeout 900 python -m pytest tests/test_gpu_fused_grad.py -x -q 2>&1 | tail -15 > gpurun_out/fused/tests.log
timeout 600 python tools/bench_fused_grad.py > gpurun_out/fused/c2.json 2> gpurun_out/fused/c2.err
timeout 600 python tools/bench_fused_grad.py 64 25557032 7 1 > gpurun_out/fused/c2_stale.json 2>> gpurun_out/fused/c2.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/fused/launches.csv python tools/bench_fused_grad.py 64 25557032 1 > gpurun_out/fused/ncu.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_objectives.py tests/test_gpu_simulation.py tests/test_gpu_acceptance.py -x -q 2>&1 | tail -5 > gpurun_out/fused/tests_sim.log
cat gpurun_out/fused/tests.log gpurun_out/fused/c2.json gpurun_out/fused/c2_stale.json gpurun_out/fused/tests_sim.log
