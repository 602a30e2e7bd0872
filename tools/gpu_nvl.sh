cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --nproc-per-node 2"
timeout 600 $TR --master-port 29931 bench.py --gpus 2 --steps 30 --warmup 5 --no-cpu --no-e2e --layout learner > gpurun_out/nvl_learner.log 2>&1
timeout 600 $TR --master-port 29932 bench.py --gpus 2 --steps 30 --warmup 5 --no-cpu --no-e2e --layout position > gpurun_out/nvl_position.log 2>&1
