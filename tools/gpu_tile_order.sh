#!/bin/bash
# mix kernel tile order: strided (default) vs blocked (RINGMIX_TILE_ORDER=blocked)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
out=gpurun_out/${1:-tile_order}; mkdir -p $out
RINGMIX_TILE_ORDER=blocked timeout 600 python -m pytest tests/test_gpu_mix.py tests/test_gpu_simulation.py -q -x -p no:cacheprovider > $out/pytest_blocked.log 2>&1; echo rc=$? >> $out/pytest_blocked.log
P="timeout 300 python tools/probe_mix.py"
for rep in 1 2 3; do
  for o in strided blocked; do
    RINGMIX_TILE_ORDER=$o $P --reps 4 > $out/c2_${o}_$rep.jsonl 2>&1
    RINGMIX_TILE_ORDER=$o $P --L 128 --d 43154944 --n 10 > $out/c3_${o}_$rep.jsonl 2>&1
    RINGMIX_TILE_ORDER=$o $P --reps 4 --mode mean > $out/c4_${o}_$rep.jsonl 2>&1
  done
done
tail -1 $out/pytest_blocked.log
python - <<PY
import json,glob,statistics,collections
res=collections.defaultdict(list)
for f in sorted(glob.glob("$out/c*.jsonl")):
    name=f.split('/')[-1].rsplit('_',1)[0]
    for l in open(f):
        if l.startswith('{'):
            d=json.loads(l)
            if d.get('what')=='mix': res[name].append(d['GBs'])
for k in sorted(res): print(k, round(statistics.median(res[k])), round(max(res[k])), len(res[k]))
PY
