cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
timeout 600 python -m pytest tests/test_gpu_multi.py tests/test_gpu_shard.py -x -q -p no:cacheprovider > gpurun_out/pytest_multi.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_multi.log
timeout 300 python -m torch.distributed.run --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29917 tools/dist_check.py > gpurun_out/dist_check.log 2>&1
for C in nvls nccl; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29920 bench.py --gpus $N --steps 50 --warmup 5 --no-cpu --no-e2e --layout learner --strategy d1d --d1d-collective $C > gpurun_out/d1d_${C}_n$N.log 2>&1
done
