#!/bin/bash
# A/B: pre-shifted staged-row offsets for one-box ring tiles (default) vs generic indexing
set -u
cd "${GRAFT_REPO_ROOT:-/root/repo}"
out=gpurun_out/${1:-mix_pre}; mkdir -p $out
L=paper_2002_01119_b200/lib
cp $L/libringmix_b200.so /tmp/main.so
timeout 900 python -m pytest tests/test_gpu_mix.py tests/test_gpu_simulation.py tests/test_gpu_fuzz.py tests/test_gpu_fullsize.py -q -x -p no:cacheprovider > $out/pytest.log 2>&1; echo rc=$? >> $out/pytest.log
P="timeout 300 python tools/probe_mix.py"
for rep in 1 2 3; do
  for v in main nopre; do
    if [ $v = main ]; then cp /tmp/main.so $L/libringmix_b200.so; else cp $L/variants/libringmix_b200_$v.so $L/libringmix_b200.so; fi
    $P --reps 4 > $out/c2_${v}_$rep.jsonl 2>&1
    $P --L 128 --d 43154944 --n 10 > $out/c3_${v}_$rep.jsonl 2>&1
    $P --L 16 --d 1048576 --n 300 > $out/c1_${v}_$rep.jsonl 2>&1
    $P --reps 2 --dtype bfloat16 > $out/c2bf_${v}_$rep.jsonl 2>&1
  done
done
cp /tmp/main.so $L/libringmix_b200.so
tail -2 $out/pytest.log
for f in $out/c*.jsonl; do echo "$f $(tail -1 $f | cut -c1-200)"; done
