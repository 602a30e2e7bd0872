cd $GRAFT_REPO_ROOT
O=gpurun_out/n2_sweep; mkdir -p $O
for rep in 1 2; do
for cfg in "3 64" "3 72" "4 56"; do
  set -- $cfg
  RINGMIX_SHARD_STAGES=$1 RINGMIX_SHARD_STAGE_KB=$2 timeout 300 python bench.py --gpus 2 --no-extras --no-e2e --steps 100 > $O/pos_n2_s$1_kb$2_r$rep.log 2>&1
done
done
for f in $O/*.log; do python -c "
import json,sys
l=[x for x in open('$f') if x.startswith('{')]
print('$f', json.loads(l[-1])['value']/1e9 if l else open('$f').read()[-300:])
"; done
