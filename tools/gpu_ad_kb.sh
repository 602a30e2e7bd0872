#!/bin/bash
# fixed ring learner-sharded: stage target 64 KB (default) vs 72 / 80 KB (3 stages)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/${1:-ad_kb}; mkdir -p $O
n=$(nvidia-smi -L | wc -l)
B="timeout 300 python bench.py --gpus $n --no-extras --no-e2e --steps 100 --strategy adpsgd_fixed"
for rep in 1 2; do
  $B > $O/kb64_r$rep.log 2>&1
  RINGMIX_SHARD_STAGE_KB=72 $B > $O/kb72_r$rep.log 2>&1
  RINGMIX_SHARD_STAGE_KB=80 $B > $O/kb80_r$rep.log 2>&1
done
for f in $O/*.log; do python -c "
import json
l=[x for x in open('$f') if x.startswith('{')]
print('$f', round(json.loads(l[-1])['value']/1e9,1) if l else open('$f').read()[-300:])
"; done
