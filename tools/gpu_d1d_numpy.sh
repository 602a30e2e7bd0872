#!/bin/bash
# numpy-order learner-sharded D1D: multi-GPU tests, dist_check, D1D bench line, trainer probe
cd "${GRAFT_REPO_ROOT:-/root/repo}"
o=gpurun_out/${1:-d1d_numpy}; mkdir -p $o
n=$(nvidia-smi -L | wc -l)
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 900 python -m pytest tests/test_gpu_multi.py -x -q -p no:cacheprovider > $o/pytest_multi.log 2>&1; echo "rc=$?" >> $o/pytest_multi.log
timeout 600 $TR --nproc-per-node $n --master-port 29851 tools/dist_check.py > $o/dist_check_n$n.log 2>&1; echo "rc=$?" >> $o/dist_check_n$n.log
timeout 600 python bench.py --gpus $n --strategy d1d --no-extras --no-e2e > $o/bench_d1d_n$n.log 2>&1
RINGMIX_D1D_NUMPY_ORDER=1 timeout 600 python bench.py --gpus $n --strategy d1d --no-extras --no-e2e > $o/bench_d1d_n${n}_numpy.log 2>&1
RINGMIX_D1D_NUMPY_ORDER=0 timeout 600 python bench.py --gpus $n --strategy d1d --no-extras --no-e2e > $o/bench_d1d_n${n}_legacy.log 2>&1
RINGMIX_D1D_TRAIN_CTAS_LIST="4,0,1" timeout 900 $TR --nproc-per-node $n --master-port 29852 tools/d1d_train_probe.py > $o/d1d_train_n$n.json 2> $o/d1d_train_n$n.err
tail -n 2 $o/pytest_multi.log; grep -h "{" $o/dist_check_n$n.log; cat $o/d1d_train_n$n.json
for f in $o/bench_d1d*.log; do python -c "
import json
l=[x for x in open('$f') if x.startswith('{')]
print('$f', round(json.loads(l[-1])['value']/1e9,1) if l else open('$f').read()[-400:])
"; done
