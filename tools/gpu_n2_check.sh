# quick 2-GPU re-check of the bench layouts (driver-like default, learner / position RAD, fused D1D)
cd $GRAFT_REPO_ROOT
O=gpurun_out/n2_final; mkdir -p $O
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --nproc-per-node 2"
timeout 600 $TR --master-port 29811 bench.py --gpus 2 > $O/drv_ours_n2.log 2>&1
for lay in learner position; do timeout 600 $TR --master-port 29812 bench.py --gpus 2 --steps 50 --warmup 5 --no-cpu --no-e2e --layout $lay > $O/rad_${lay}_n2.log 2>&1; done
timeout 600 $TR --master-port 29813 bench.py --gpus 2 --steps 50 --warmup 5 --no-cpu --no-e2e --layout learner --strategy d1d > $O/d1d_fused_n2.log 2>&1
