cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
run() { timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29920 bench.py --gpus $N --steps 50 --warmup 5 --no-cpu --no-e2e --layout learner --strategy d1d --d1d-collective nvls --d1d-chunk-cols $1 2>&1 | grep -o '"ms_per_step": [0-9.]*' | sed "s/^/$1 $RINGMIX_D1D_CTAS /" >> gpurun_out/d1d_pipe_n$N.log; }
: > gpurun_out/d1d_pipe_n$N.log
run 0
for C in "4,2,2" "8,2,2" "4,2,1" "4,1,2" "8,3,0"; do export RINGMIX_D1D_CTAS=$C; run 4194304; run 8388608; done
