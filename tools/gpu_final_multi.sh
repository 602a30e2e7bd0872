# round-end multi-GPU pass (gpurun --gpus 4)
cd $GRAFT_REPO_ROOT
O=gpurun_out/final_multi; mkdir -p $O
free -g > $O/free.txt 2>&1; nproc >> $O/free.txt; nvidia-smi topo -m > $O/topo.txt 2>&1
N=$(nvidia-smi -L | wc -l)
timeout 900 python -m pytest tests/test_gpu_multi.py tests/test_gpu_shard.py -q -p no:cacheprovider > $O/pytest_multi.log 2>&1; echo "rc=$?" >> $O/pytest_multi.log
timeout 300 python -m torch.distributed.run --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29917 tools/dist_check.py > $O/dist_check.log 2>&1; echo "rc=$?" >> $O/dist_check.log
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
# driver-like: default arms at n = 1, 2, 4
( time timeout 900 python bench.py ) > $O/drv_ours_n1.log 2>&1
( time timeout 900 python bench.py --impl reference ) > $O/drv_ref_n1.log 2>&1
for n in 2 4; do
  ( time timeout 900 $TR --nproc-per-node $n --master-port $((29800+n)) bench.py --gpus $n ) > $O/drv_ours_n$n.log 2>&1
  ( time timeout 900 $TR --nproc-per-node $n --master-port $((29810+n)) bench.py --impl reference --gpus $n ) > $O/drv_ref_n$n.log 2>&1
done
# layouts (C2 problem fixed = strong), n = 2 and 4
for n in 2 4; do
  P=$((29900+n))
  timeout 600 $TR --nproc-per-node $n --master-port $P bench.py --gpus $n --steps 50 --warmup 5 --no-cpu --no-e2e --scaling strong > $O/coord_strong_n$n.log 2>&1
  timeout 600 $TR --nproc-per-node $n --master-port $P bench.py --gpus $n --steps 50 --warmup 5 --no-cpu --no-e2e --layout learner --strategy adpsgd_fixed > $O/ad_learner_n$n.log 2>&1
  timeout 600 $TR --nproc-per-node $n --master-port $P bench.py --gpus $n --steps 50 --warmup 5 --no-cpu --no-e2e --layout learner > $O/rad_learner_n$n.log 2>&1
  timeout 600 $TR --nproc-per-node $n --master-port $P bench.py --gpus $n --steps 50 --warmup 5 --no-cpu --no-e2e --layout position > $O/rad_position_n$n.log 2>&1
  timeout 600 $TR --nproc-per-node $n --master-port $P bench.py --gpus $n --steps 50 --warmup 5 --no-cpu --no-e2e --layout learner --strategy d1d > $O/d1d_fused_n$n.log 2>&1
  timeout 600 $TR --nproc-per-node $n --master-port $P bench.py --gpus $n --steps 50 --warmup 5 --no-cpu --no-e2e --layout learner --strategy d1d --d1d-collective nvls > $O/d1d_nvls_n$n.log 2>&1
  timeout 600 $TR --nproc-per-node $n --master-port $P bench.py --gpus $n --steps 50 --warmup 5 --no-cpu --no-e2e --layout learner --strategy d1d --d1d-chunk-cols 0 > $O/d1d_nvls1_n$n.log 2>&1
  timeout 600 $TR --nproc-per-node $n --master-port $P bench.py --gpus $n --steps 50 --warmup 5 --no-cpu --no-e2e --layout learner --strategy d1d --d1d-collective nccl > $O/d1d_nccl_n$n.log 2>&1
done
for SP in "35,10" "30,5" "25,10"; do
  RINGMIX_D1D_FUSED_SPLIT=$SP timeout 600 $TR --nproc-per-node 4 --master-port 29950 bench.py --gpus 4 --steps 50 --warmup 5 --no-cpu --no-e2e --layout learner --strategy d1d > $O/d1d_fused_split_${SP/,/_}_n4.log 2>&1
done
echo done > $O/done.txt
