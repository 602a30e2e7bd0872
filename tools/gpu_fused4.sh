cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --nproc-per-node $N"
timeout 300 $TR --master-port 29917 tools/dist_check.py > gpurun_out/fused_check4.log 2>&1; echo "rc=$?" >> gpurun_out/fused_check4.log
: > gpurun_out/fused_bench4.log
timeout 300 $TR --master-port 29920 bench.py --gpus $N --steps 50 --warmup 5 --no-cpu --no-e2e --layout learner --strategy d1d --d1d-collective nvls 2>&1 | grep -o '"ms_per_step": [0-9.]*' | sed "s/^/nvls /" >> gpurun_out/fused_bench4.log
for SP in "30,10" "25,10" "30,15" "35,15"; do
RINGMIX_D1D_FUSED_SPLIT=$SP timeout 300 $TR --master-port 29921 bench.py --gpus $N --steps 50 --warmup 5 --no-cpu --no-e2e --layout learner --strategy d1d --d1d-collective fused 2>&1 | grep -o '"ms_per_step": [0-9.]*' | sed "s/^/fused split=$SP /" >> gpurun_out/fused_bench4.log
done
