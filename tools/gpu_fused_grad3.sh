#!/bin/bash
# fused gradient+mix: tests, C2 sync/stale timings, then the RM_FAST_F2D variant
cd "${GRAFT_REPO_ROOT:-/root/repo}"
o=gpurun_out/${1:-fused9}
mkdir -p $o
timeout 900 python -m pytest tests/test_gpu_fused_grad.py -x -q 2>&1 | tail -3 > $o/tests.log
timeout 600 python tools/bench_fused_grad.py > $o/c2.json 2> $o/c2.err
timeout 600 python tools/bench_fused_grad.py 64 25557032 7 1 > $o/c2_stale.json 2>> $o/c2.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  -k regex:mix_tma --log-file $o/launches.csv python tools/bench_fused_grad.py 64 25557032 1 > $o/ncu.log 2>&1
for v in paper_2002_01119_b200/lib/variants/*.so; do
  [ -e "$v" ] || continue
  n=$(basename $v .so)
  cp paper_2002_01119_b200/lib/libringmix_b200.so /tmp/base.so
  cp $v paper_2002_01119_b200/lib/libringmix_b200.so
  timeout 600 python tools/bench_fused_grad.py > $o/c2_$n.json 2>> $o/c2.err
  timeout 600 python tools/bench_fused_grad.py 64 25557032 7 1 > $o/c2_stale_$n.json 2>> $o/c2.err
  cp /tmp/base.so paper_2002_01119_b200/lib/libringmix_b200.so
done
cd $o; for f in tests.log c2*.json; do echo "== $f"; cat $f; done
