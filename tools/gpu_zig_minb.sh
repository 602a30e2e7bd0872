#!/bin/bash
# speculative kernel occupancy: build variants with __launch_bounds__(128, MINB)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
o=gpurun_out/${1:-zig_minb}; mkdir -p $o
L=paper_2002_01119_b200/lib
cp $L/libringmix_b200.so /tmp/main.so
for v in main mb8 mb9 main mb8 mb9; do
  if [ $v = main ]; then cp /tmp/main.so $L/libringmix_b200.so; else cp $L/variants/libringmix_b200_$v.so $L/libringmix_b200.so; fi
  timeout 300 python -c "
import sys; sys.path.insert(0,'tools'); import bench_grad as b
b.main(64, 25_557_032, reps=9)" >> $o/grad_$v.log 2>&1
done
cp $L/variants/libringmix_b200_mb8.so $L/libringmix_b200.so
timeout 600 python -m pytest tests/test_gpu_objectives.py -q -x -p no:cacheprovider -k "normal or gradients" > $o/pytest_mb8.log 2>&1; echo "rc=$?" >> $o/pytest_mb8.log
cp /tmp/main.so $L/libringmix_b200.so
tail -2 $o/pytest_mb8.log; for f in $o/grad_*.log; do echo "== $f"; cat $f | python -c "import sys,json; [print(json.loads(l)['grad_ms']) for l in sys.stdin if l.startswith('{')]"; done
