#!/bin/bash
# A/B: fp32->fp64 widening by integer re-biasing (RM_FAST_F2D) vs F2F, C2/C3/C1 + parity tests
set -u
out=gpurun_out/mix_ab4; mkdir -p $out
L=paper_2002_01119_b200/lib
cp $L/libringmix_b200.so $L/libringmix_b200.so.orig
P="timeout 300 python tools/probe_mix.py"
for rep in 1 2; do
  for v in orig f2d; do
    if [ $v = orig ]; then cp $L/libringmix_b200.so.orig $L/libringmix_b200.so; else cp $L/variants/libringmix_b200_$v.so $L/libringmix_b200.so; fi
    $P --reps 4 > $out/c2_${v}_$rep.jsonl 2>&1
    $P --L 128 --d 43154944 --n 10 > $out/c3_${v}_$rep.jsonl 2>&1
    $P --L 16 --d 1048576 --n 300 > $out/c1_${v}_$rep.jsonl 2>&1
  done
done
cp $L/variants/libringmix_b200_f2d.so $L/libringmix_b200.so
timeout 600 python -m pytest tests/test_gpu_mix.py tests/test_gpu_simulation.py -q -x > $out/pytest_f2d.log 2>&1; echo rc=$? >> $out/pytest_f2d.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:mix_tma -s 6 -c 1 -o $out/mix_c2_f2d python tools/probe_mix.py --reps 1 --n 3 > $out/ncu_f2d.log 2>&1
cp $L/libringmix_b200.so.orig $L/libringmix_b200.so
tail -2 $out/pytest_f2d.log
