# fused D1D: column-chunk size sweep (learner-sharded, all GPUs of the box)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --nproc-per-node $N"
: > gpurun_out/fused_chunk.log
for CH in 2097152 1048576 524288 4194304; do
RINGMIX_D1D_FUSED_CHUNK=$CH timeout 300 $TR --master-port 29921 bench.py --gpus $N --steps 50 --warmup 5 --no-cpu --no-e2e --layout learner --strategy d1d 2>&1 | grep -o '"ms_per_step": [0-9.]*' | sed "s/^/chunk=$CH /" >> gpurun_out/fused_chunk.log
done
