#!/bin/bash
# ring tiles: one 512-thread CTA per SM (default) vs one 1024-thread CTA (RINGMIX_RING_NT=1024)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
out=gpurun_out/${1:-ring_nt}; mkdir -p $out
RINGMIX_RING_NT=1024 timeout 600 python -m pytest tests/test_gpu_mix.py -q -x -p no:cacheprovider > $out/pytest_1024.log 2>&1; echo rc=$? >> $out/pytest_1024.log
P="timeout 300 python tools/probe_mix.py"
for rep in 1 2 3; do
  for nt in 512 1024; do
    RINGMIX_RING_NT=$nt $P --reps 4 > $out/c2_${nt}_$rep.jsonl 2>&1
    RINGMIX_RING_NT=$nt $P --L 128 --d 43154944 --n 10 > $out/c3_${nt}_$rep.jsonl 2>&1
    RINGMIX_RING_NT=$nt $P --reps 2 --dtype bfloat16 > $out/c2bf_${nt}_$rep.jsonl 2>&1
  done
done
tail -1 $out/pytest_1024.log
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
