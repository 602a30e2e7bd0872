cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
nvidia-smi topo -m > gpurun_out/topo_n$N.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_shard.py tests/test_gpu_multi.py -x -q -p no:cacheprovider > gpurun_out/pytest_multi_n$N.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_multi_n$N.log
for n in 1 2 4 8; do
  [ $n -gt $N ] && continue
  for LAY in coord learner; do
    [ $n -eq 1 ] && [ $LAY = learner ] && continue
    timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29700+n)) bench.py --gpus $n --steps 50 --warmup 5 --no-cpu --no-e2e --layout $LAY > gpurun_out/scale_${LAY}_n$n.log 2>&1; echo "rc=$?" >> gpurun_out/scale_${LAY}_n$n.log
  done
  [ $n -gt 1 ] && timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29720+n)) bench.py --gpus $n --steps 50 --warmup 5 --no-cpu --no-e2e --layout learner --strategy d1d > gpurun_out/scale_d1d_learner_n$n.log 2>&1
  [ $n -gt 1 ] && timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29740+n)) bench.py --gpus $n --steps 50 --warmup 5 --no-cpu --no-e2e --layout learner --strategy adpsgd_fixed > gpurun_out/scale_ad_learner_n$n.log 2>&1
done
exit 0
