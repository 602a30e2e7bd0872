#!/bin/bash
# A/B round 2 (b): ring-kernel variants (staged TMA with unroll 1/2/4, direct-load 'ldg'),
# PDL on/off, C1 bench with CUDA graph; new GPU tests.
set -u
out=gpurun_out/mix_ab3; mkdir -p $out
L=paper_2002_01119_b200/lib
cp $L/libringmix_b200.so $L/libringmix_b200.so.orig
P="timeout 300 python tools/probe_mix.py"
run_set() {   # $1 = tag, env already set by caller
  $P --reps 4 > $out/c2_$1.jsonl 2>&1
  $P --L 128 --d 43154944 --n 10 > $out/c3_$1.jsonl 2>&1
  $P --L 16 --d 1048576 --n 300 > $out/c1_$1.jsonl 2>&1
  $P --dtype bfloat16 > $out/c2bf16_$1.jsonl 2>&1
}
run_set base
RINGMIX_RING_IMPL=ldg run_set ldg
RINGMIX_PDL=1 run_set pdl
for v in u1 u4; do
  cp $L/variants/libringmix_b200_$v.so $L/libringmix_b200.so
  run_set $v
done
cp $L/libringmix_b200.so.orig $L/libringmix_b200.so
timeout 300 python bench.py --learners 16 --dim 1048576 --no-cpu --no-e2e --steps 400 > $out/bench_c1_graph.log 2>&1
timeout 300 python bench.py --learners 16 --dim 1048576 --no-cpu --no-e2e --steps 400 --graph off > $out/bench_c1_nograph.log 2>&1
RINGMIX_RING_IMPL=ldg timeout 300 python bench.py --learners 16 --dim 1048576 --no-cpu --no-e2e --steps 400 > $out/bench_c1_graph_ldg.log 2>&1
timeout 600 python bench.py --no-cpu --no-e2e --no-extras > $out/bench_c2.log 2>&1
RINGMIX_RING_IMPL=ldg timeout 600 python bench.py --no-cpu --no-e2e --no-extras > $out/bench_c2_ldg.log 2>&1
RINGMIX_RING_IMPL=ldg timeout 600 python -m pytest tests/test_gpu_mix.py -q -x > $out/pytest_ldg.log 2>&1; echo rc=$? >> $out/pytest_ldg.log
timeout 600 python -m pytest tests/test_gpu_mix.py tests/test_gpu_simulation.py tests/test_gpu_dL.py tests/test_gpu_perm.py -q -x > $out/pytest.log 2>&1; echo rc=$? >> $out/pytest.log
for f in $out/*.log; do echo "== $f"; tail -3 $f | cut -c1-300; done
