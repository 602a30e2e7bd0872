# BASELINE config 3 (RAD, 128 learners x 43,154,944) across GPUs: learner-sharded (pull, position)
# and coordinate stripes (strong), n = 2 and 4
cd $GRAFT_REPO_ROOT
O=gpurun_out/c3_multi; mkdir -p $O
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
for n in 2 4; do
  for LAY in learner position; do
    timeout 600 $TR --nproc-per-node $n --master-port 29960 bench.py --gpus $n --steps 20 --warmup 3 --no-cpu --no-e2e --learners 128 --dim 43154944 --layout $LAY > $O/c3_${LAY}_n$n.log 2>&1
  done
  timeout 600 $TR --nproc-per-node $n --master-port 29961 bench.py --gpus $n --steps 20 --warmup 3 --no-cpu --no-e2e --learners 128 --dim 43154944 --scaling strong > $O/c3_coord_strong_n$n.log 2>&1
done
timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu --no-e2e --learners 128 --dim 43154944 > $O/c3_n1.log 2>&1
