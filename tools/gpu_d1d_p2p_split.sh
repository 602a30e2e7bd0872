#!/bin/bash
# numpy-order D1D over peer tables at n = 4: role splits of the fused kernel (partial, reduce %)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
o=gpurun_out/${1:-d1d_p2p_split}; mkdir -p $o
n=$(nvidia-smi -L | wc -l)
for sp in 30,10 25,25 20,40 15,55 30,30; do
  for occ in 4 2; do
    RINGMIX_D1D_FUSED_OCC=$occ RINGMIX_D1D_FUSED_SPLIT=$sp RINGMIX_D1D_NUMPY_ORDER=1 timeout 300 python bench.py --gpus $n --strategy d1d --no-extras --no-e2e --steps 50 > $o/np_${sp/,/_}_o$occ.log 2>&1
  done
done
RINGMIX_D1D_NUMPY_ORDER=0 RINGMIX_SYM_P2P=1 timeout 300 python bench.py --gpus $n --strategy d1d --no-extras --no-e2e --steps 50 > $o/legacy_p2p.log 2>&1
RINGMIX_D1D_NUMPY_ORDER=0 timeout 300 python bench.py --gpus $n --strategy d1d --no-extras --no-e2e --steps 50 > $o/legacy_nvls.log 2>&1
for f in $o/*.log; do python -c "
import json
l=[x for x in open('$f') if x.startswith('{')]
print('$f', round(json.loads(l[-1])['value']/1e9,1) if l else open('$f').read()[-300:])
"; done
