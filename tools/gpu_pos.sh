cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
timeout 900 python -m pytest tests/test_gpu_shard.py tests/test_gpu_multi.py -x -q -p no:cacheprovider > gpurun_out/pytest_pos.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_pos.log
timeout 300 python -m torch.distributed.run --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29917 tools/dist_check.py > gpurun_out/dist_check.log 2>&1
for n in 2 4; do for LAY in learner position; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29940+n)) bench.py --gpus $n --steps 50 --warmup 5 --no-cpu --no-e2e --layout $LAY > gpurun_out/rad_${LAY}_n$n.log 2>&1
done; done
