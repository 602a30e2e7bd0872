cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --nproc-per-node $N"
timeout 600 python -m pytest tests/test_gpu_shard.py tests/test_gpu_multi.py -q -p no:cacheprovider > gpurun_out/ss_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/ss_pytest.log
timeout 300 $TR --master-port 29917 tools/dist_check.py > gpurun_out/ss_check.log 2>&1; echo "rc=$?" >> gpurun_out/ss_check.log
: > gpurun_out/ss_bench.log
for LAY in learner position; do for SS in 1 0; do
RINGMIX_STEP_SYNC=$SS timeout 300 $TR --master-port 29920 bench.py --gpus $N --steps 50 --warmup 5 --no-cpu --no-e2e --layout $LAY 2>&1 | grep '^{' | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('$LAY', 'sync=$SS', d['ms_per_step'], d.get('step_ordering'), d['gpu_launches_detail'])" >> gpurun_out/ss_bench.log 2>&1
done; done
