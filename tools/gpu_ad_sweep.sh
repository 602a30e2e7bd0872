#!/bin/bash
# fixed ring (AD-PSGD), learners sharded (pull kernel, only the 2 boundary rows cross GPUs):
# stage count / size sweep at C2 on all GPUs of the box, against the no-communication stripes
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/${1:-ad_sweep}; mkdir -p $O
n=$(nvidia-smi -L | wc -l)
B="timeout 300 python bench.py --gpus $n --no-extras --no-e2e --steps 100"
$B --strategy adpsgd_fixed > $O/ad_default.log 2>&1
for cfg in "3 32" "4 48" "6 32" "4 32" "2 96"; do
  set -- $cfg
  RINGMIX_SHARD_STAGES=$1 RINGMIX_SHARD_STAGE_KB=$2 $B --strategy adpsgd_fixed > $O/ad_s$1_kb$2.log 2>&1
done
$B --strategy adpsgd_fixed --layout coord --scaling strong > $O/ad_coord_strong.log 2>&1
for f in $O/*.log; do python -c "
import json
l=[x for x in open('$f') if x.startswith('{')]
d=json.loads(l[-1]) if l else None
print('$f', round(d['value']/1e9,1) if d else open('$f').read()[-300:], d and round(d['roofline']['frac'],3), d and round(d['ms_per_step'],3))
"; done
