#!/bin/bash
# generator scratch: lane-interleaved quads (default) vs contiguous blocks (variant noil):
# normal / gradient / fused-step parity tests, C2 gradient and fused-step timing
cd "${GRAFT_REPO_ROOT:-/root/repo}"
o=gpurun_out/${1:-zig_il}; mkdir -p $o
L=paper_2002_01119_b200/lib
cp $L/libringmix_b200.so /tmp/main.so
timeout 900 python -m pytest tests/test_gpu_objectives.py tests/test_gpu_fused_grad.py -q -x -p no:cacheprovider > $o/pytest.log 2>&1; echo "rc=$?" >> $o/pytest.log
for v in main noil main noil; do
  if [ $v = main ]; then cp /tmp/main.so $L/libringmix_b200.so; else cp $L/variants/libringmix_b200_$v.so $L/libringmix_b200.so; fi
  timeout 300 python -c "
import sys; sys.path.insert(0,'tools'); import bench_grad as b
b.main(64, 25_557_032, reps=9)" >> $o/grad_$v.log 2>&1
  timeout 300 python tools/bench_fused_grad.py >> $o/fused_$v.log 2>&1
done
cp /tmp/main.so $L/libringmix_b200.so
tail -2 $o/pytest.log; for f in $o/grad_*.log $o/fused_*.log; do echo "== $f"; tail -4 $f; done
