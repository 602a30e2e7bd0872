#!/bin/bash
# ncu --set full of the fused gradient+mix kernel (sync and stale Phi) at C2
cd "${GRAFT_REPO_ROOT:-/root/repo}"
tag=${1:-x}
mkdir -p gpurun_out/fused_ncu
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"mix_tma_kernel" -s 3 -c 1 \
  -o gpurun_out/fused_ncu/$tag python tools/bench_fused_grad.py 64 25557032 1 > gpurun_out/fused_ncu/ncu_$tag.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"mix_tma_kernel" -s 3 -c 1 \
  -o gpurun_out/fused_ncu/${tag}_stale python tools/bench_fused_grad.py 64 25557032 1 1 > gpurun_out/fused_ncu/ncu_${tag}_stale.log 2>&1
tail -2 gpurun_out/fused_ncu/ncu_$tag.log gpurun_out/fused_ncu/ncu_${tag}_stale.log
