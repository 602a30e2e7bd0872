#!/bin/bash
# A/B round 2: unroll variants, PDL on/off, C1 bench with CUDA graph, triad ceiling.
set -u
out=gpurun_out/mix_ab2; mkdir -p $out
L=paper_2002_01119_b200/lib
cp $L/libringmix_b200.so $L/libringmix_b200.so.orig
P="timeout 300 python tools/probe_mix.py"
$P --ceiling --reps 3 > $out/ceiling.jsonl 2>&1
for v in u1 u2 u4; do
  cp $L/variants/libringmix_b200_$v.so $L/libringmix_b200.so
  $P --reps 4 > $out/c2_$v.jsonl 2>&1
  $P --L 128 --d 43154944 --n 10 > $out/c3_$v.jsonl 2>&1
  $P --L 16 --d 1048576 --n 300 > $out/c1_$v.jsonl 2>&1
  RINGMIX_PDL=0 $P --L 16 --d 1048576 --n 300 > $out/c1_${v}_nopdl.jsonl 2>&1
  $P --dtype bfloat16 > $out/c2bf16_$v.jsonl 2>&1
done
cp $L/libringmix_b200.so.orig $L/libringmix_b200.so
timeout 300 python bench.py --learners 16 --dim 1048576 --no-cpu --no-e2e --steps 400 > $out/bench_c1_graph.log 2>&1
timeout 300 python bench.py --learners 16 --dim 1048576 --no-cpu --no-e2e --steps 400 --graph off > $out/bench_c1_nograph.log 2>&1
RINGMIX_PDL=0 timeout 300 python bench.py --learners 16 --dim 1048576 --no-cpu --no-e2e --steps 400 > $out/bench_c1_graph_nopdl.log 2>&1
timeout 600 python -m pytest tests/test_gpu_mix.py tests/test_gpu_simulation.py tests/test_gpu_dL.py tests/test_gpu_perm.py -q -x > $out/pytest.log 2>&1; echo rc=$? >> $out/pytest.log
timeout 1200 python -m pytest tests/test_gpu_reference_suite.py -q -x -k "not acceptance" > $out/pytest_refsuite.log 2>&1; echo rc=$? >> $out/pytest_refsuite.log
timeout 300 python tools/bench_trace.py > $out/bench_trace.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:trace_stats_tma -s 2 -c 1 -o $out/trace_c2 python tools/bench_trace.py > $out/ncu_trace.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:mix_tma -s 6 -c 1 -o $out/mix_c2 python tools/probe_mix.py --reps 1 --n 3 > $out/ncu_mix.log 2>&1
for f in $out/*.jsonl $out/*.log; do echo "== $f"; tail -5 $f; done
