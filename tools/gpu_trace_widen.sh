#!/bin/bash
# trace tile kernel: F2F vs integer widening (build variants), parity + C2/C3 timing
cd "${GRAFT_REPO_ROOT:-/root/repo}"
o=gpurun_out/${1:-trace_widen}; mkdir -p $o
L=paper_2002_01119_b200/lib
cp $L/libringmix_b200.so /tmp/main.so
for v in main tw1 tw2 tw3 main tw3; do
  if [ $v = main ]; then cp /tmp/main.so $L/libringmix_b200.so; else cp $L/variants/libringmix_b200_$v.so $L/libringmix_b200.so; fi
  timeout 300 python tools/bench_trace.py --reps 10 2>&1 | grep -v exact_order | head -3 > $o/$v.jsonl
  timeout 300 python -m pytest tests/test_gpu_objectives.py -q -x -k trace -p no:cacheprovider 2>&1 | tail -1 >> $o/$v.jsonl
done
cp /tmp/main.so $L/libringmix_b200.so
for f in $o/*.jsonl; do echo "== $f"; cat $f | python -c "
import sys,json
for l in sys.stdin:
  l=l.strip()
  if l.startswith('{'):
    d=json.loads(l); print(d['L'], d['dtype'], d['tile']['ms'], d['tile']['frac'])
  else: print(l)"; done
