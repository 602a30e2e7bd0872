#!/bin/bash
# D1D training step across GPUs: serial vs overlapped (ShardedD1DTrainer) with CTA caps, C4 shapes
cd "${GRAFT_REPO_ROOT:-/root/repo}"
o=gpurun_out/${1:-d1d_train}
mkdir -p $o
n=$(nvidia-smi -L | wc -l)
timeout 600 python -m pytest tests/test_gpu_objectives.py -x -q -k sharded 2>&1 | tail -2 > $o/tests.log
RINGMIX_D1D_TRAIN_CTAS_LIST="${CAPS:-1,0,1;2,0,1;4,0,1}" timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
  --master-port 29531 tools/d1d_train_probe.py > $o/n$n.json 2> $o/n$n.err
cat $o/tests.log $o/n$n.json; tail -5 $o/n$n.err
