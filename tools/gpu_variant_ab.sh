#!/bin/bash
# A/B of the built library variants (paper_2002_01119_b200/lib/variants/*.so) against the
# product library: mix parity tests + bench.py N=1 (no extras), alternating twice
cd "${GRAFT_REPO_ROOT:-/root/repo}"
o=gpurun_out/${1:-variant_ab}; mkdir -p $o
tests=${2:-tests/test_gpu_mix.py}
cp paper_2002_01119_b200/lib/libringmix_b200.so /tmp/base.so
for rep in 1 2; do
  for v in base paper_2002_01119_b200/lib/variants/*.so; do
    n=$(basename $v .so)
    if [ "$v" = base ]; then cp /tmp/base.so paper_2002_01119_b200/lib/libringmix_b200.so
    else cp $v paper_2002_01119_b200/lib/libringmix_b200.so; fi
    if [ $rep = 1 ]; then
      timeout 900 python -m pytest $tests -x -q -p no:cacheprovider 2>&1 | tail -1 > $o/tests_$n.log
    fi
    timeout 600 python bench.py --no-extras --steps 100 --warmup 5 > $o/bench_${n}_$rep.json 2> $o/bench_${n}_$rep.err
  done
done
cp /tmp/base.so paper_2002_01119_b200/lib/libringmix_b200.so
cd $o; for f in tests_*.log; do echo "$f: $(cat $f)"; done
for f in bench_*.json; do python -c "import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', round(d['value']/1e9,1), d['roofline']['frac'], d['roofline']['avg_launch_ms'])"; done
