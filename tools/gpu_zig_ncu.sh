#!/bin/bash
# ncu --set full of the speculative ziggurat kernel at C2 (one launch)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
o=gpurun_out/zig_ncu; mkdir -p $o
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"zig_spec_kernel" -s 2 -c 1 \
  -o $o/${1:-spec} python tools/bench_fused_grad.py 64 25557032 1 > $o/ncu_${1:-spec}.log 2>&1
tail -3 $o/ncu_${1:-spec}.log
