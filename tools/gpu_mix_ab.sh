#!/bin/bash
# A/B of ring mix-kernel variants on one B200 (tools/probe_mix.py); logs -> gpurun_out/mix_ab/
set -u
out=gpurun_out/mix_ab; mkdir -p $out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $out/smi.txt
timeout 600 python -m pytest tests/test_gpu_mix.py tests/test_gpu_simulation.py tests/test_gpu_shard.py -x -q > $out/pytest.log 2>&1; echo "pytest rc=$?" >> $out/pytest.log
P="timeout 300 python tools/probe_mix.py"
$P --ceiling > $out/c2_slide.jsonl 2>&1
RINGMIX_RING_IMPL=item $P > $out/c2_item.jsonl 2>&1
RINGMIX_RING_NT=256 $P > $out/c2_slide_nt256.jsonl 2>&1
RINGMIX_RING_IMPL=item RINGMIX_RING_NT=256 $P > $out/c2_item_nt256.jsonl 2>&1
for kb in 48 56 72; do RINGMIX_STAGE_KB=$kb $P > $out/c2_slide_kb$kb.jsonl 2>&1; done
$P --fixed > $out/c2_fixed_slide.jsonl 2>&1
RINGMIX_RING_IMPL=item $P --fixed > $out/c2_fixed_item.jsonl 2>&1
$P --L 128 --d 43154944 --n 10 > $out/c3_slide.jsonl 2>&1
RINGMIX_RING_IMPL=item $P --L 128 --d 43154944 --n 10 > $out/c3_item.jsonl 2>&1
$P --L 16 --d 1048576 --n 200 > $out/c1_slide.jsonl 2>&1
RINGMIX_RING_IMPL=item $P --L 16 --d 1048576 --n 200 > $out/c1_item.jsonl 2>&1
$P --dtype bfloat16 > $out/c2bf16_slide.jsonl 2>&1
RINGMIX_RING_IMPL=item $P --dtype bfloat16 > $out/c2bf16_item.jsonl 2>&1
$P --dtype float64 --n 10 > $out/c2f64_slide.jsonl 2>&1
RINGMIX_RING_IMPL=item $P --dtype float64 --n 10 > $out/c2f64_item.jsonl 2>&1
for f in $out/*.jsonl; do echo "== $f"; cat $f; done
