#!/bin/bash
# position layout (C3 strong scaling): one 512-thread CTA per SM vs two 256-thread CTAs
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/${1:-shard_nt}; mkdir -p $O
n=$(nvidia-smi -L | wc -l)
RINGMIX_SHARD_NT=256 timeout 600 python -m pytest tests/test_gpu_emulated_world.py -q -x -p no:cacheprovider -k "position" > $O/emu256.log 2>&1; tail -1 $O/emu256.log
for rep in 1 2; do
for nt in 512 256; do
  RINGMIX_SHARD_NT=$nt timeout 300 python bench.py --gpus $n --no-extras --no-e2e --steps 100 > $O/pos_n${n}_nt${nt}_r$rep.log 2>&1
done
done
for f in $O/pos*.log; do python -c "
import json,sys
l=[x for x in open('$f') if x.startswith('{')]
print('$f', round(json.loads(l[-1])['value']/1e9,1) if l else open('$f').read()[-300:])
"; done
