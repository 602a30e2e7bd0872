#!/bin/bash
# ring mix: window path (default) vs staged triples (RINGMIX_RING_WIN=0): parity tests + bench A/B
cd "${GRAFT_REPO_ROOT:-/root/repo}"
o=gpurun_out/${1:-win_ab}; mkdir -p $o
timeout 900 python -m pytest tests/test_gpu_mix.py tests/test_gpu_simulation.py tests/test_gpu_fuzz.py tests/test_gpu_fullsize.py -q -x -p no:cacheprovider > $o/pytest.log 2>&1; echo "rc=$?" >> $o/pytest.log
for r in 1 2; do
for w in 1 0; do
  RINGMIX_RING_WIN=$w timeout 600 python bench.py --steps 100 --warmup 5 --no-cpu --no-e2e > $o/c2_w$w.r$r.json 2>/dev/null
  RINGMIX_RING_WIN=$w timeout 600 python bench.py --steps 20 --warmup 3 --learners 128 --dim 43154944 --no-cpu --no-e2e > $o/c3_w$w.r$r.json 2>/dev/null
  RINGMIX_RING_WIN=$w timeout 300 python bench.py --steps 200 --warmup 5 --learners 16 --dim 1048576 --no-cpu --no-e2e > $o/c1_w$w.r$r.json 2>/dev/null
done; done
tail -2 $o/pytest.log
for f in $o/c*.json; do python -c "
import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', round(d['value']/1e9,1), d['roofline']['frac'], d.get('clocks',{}).get('sm_mhz'))"; done
