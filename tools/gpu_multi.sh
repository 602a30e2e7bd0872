cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvidia-smi topo -m > gpurun_out/topo.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 100 --warmup 5 --cpu-seconds 3 > gpurun_out/bench_n1.log 2>&1; echo "rc=$?" >> gpurun_out/bench_n1.log
N=$(nvidia-smi -L | wc -l)
for LAY in coord learner; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29611 bench.py --gpus $N --steps 50 --warmup 5 --no-cpu --layout $LAY > gpurun_out/bench_n${N}_$LAY.log 2>&1; echo "rc=$?" >> gpurun_out/bench_n${N}_$LAY.log
done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29613 bench.py --gpus $N --steps 50 --warmup 5 --no-cpu --no-e2e --layout learner --strategy d1d > gpurun_out/bench_n${N}_learner_d1d.log 2>&1; echo "rc=$?" >> gpurun_out/bench_n${N}_learner_d1d.log
