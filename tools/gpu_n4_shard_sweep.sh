# position-layout stage sweep at n = 2 and 4 (C3), bench lines without extras / e2e
cd $GRAFT_REPO_ROOT
O=gpurun_out/n4_sweep; mkdir -p $O
for n in 4 2; do
  for cfg in "3 64" "4 48" "5 40" "2 96" "4 32" "6 32"; do
    set -- $cfg
    RINGMIX_SHARD_STAGES=$1 RINGMIX_SHARD_STAGE_KB=$2 timeout 300 python bench.py --gpus $n --no-extras --no-e2e --steps 100 > $O/pos_n${n}_s$1_kb$2.log 2>&1
  done
done
for f in $O/*.log; do python -c "
import json,sys
l=[x for x in open('$f') if x.startswith('{')]
print('$f', json.loads(l[-1])['value']/1e9 if l else open('$f').read()[-300:])
"; done
