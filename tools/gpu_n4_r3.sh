# 4-GPU pass (round 2, final session): the driver's scaling commands (both arms, N = 1, 2, 4),
# the multi-GPU tests on 4 GPUs, the D1D training step (serial vs the default concurrency) at
# N = 4 and N = 2, dist_check at n = 3 (ragged).
cd $GRAFT_REPO_ROOT
O=gpurun_out/${1:-n4_r3}; mkdir -p $O
nvidia-smi topo -m > $O/topo.txt 2>&1
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
( time timeout 900 python bench.py ) > $O/drv_ours_n1.log 2>&1
( time timeout 600 python bench.py --impl reference ) > $O/drv_ref_n1.log 2>&1
for n in 2 4; do
  ( time timeout 900 $TR --nproc-per-node $n --master-port $((29800+n)) bench.py --gpus $n ) > $O/drv_ours_n$n.log 2>&1
  ( time timeout 600 $TR --nproc-per-node $n --master-port $((29810+n)) bench.py --impl reference --gpus $n --steps 5 --warmup 3 ) > $O/drv_ref_n$n.log 2>&1
done
( time timeout 600 python bench.py --gpus 4 --strategy adpsgd_fixed --no-extras ) > $O/adpsgd_n4.log 2>&1
timeout 900 python -m pytest tests/test_gpu_multi.py tests/test_gpu_integration.py -x -q > $O/pytest_multi.log 2>&1; echo "rc=$?" >> $O/pytest_multi.log
CHK_L=10 CHK_D=4099 timeout 600 $TR --nproc-per-node 3 --master-port 29831 tools/dist_check.py > $O/dist_check_n3.log 2>&1; echo "rc=$?" >> $O/dist_check_n3.log
for n in 4 2; do
RINGMIX_D1D_TRAIN_CTAS_LIST="4,0,1" timeout 900 $TR --nproc-per-node $n --master-port $((29840+n)) tools/d1d_train_probe.py > $O/d1d_train_n$n.json 2> $O/d1d_train_n$n.err
done
tail -2 $O/*.log; cat $O/d1d_train_n*.json
for f in $O/drv_ours_n*.log; do python -c "
import json
l=[x for x in open('$f') if x.startswith('{')]
d=json.loads(l[-1]); print('$f', d['n_gpus'], round(d['value']/1e9,1), d['config'].get('layout'), {k: round(v.get('value',0)/1e9,1) for k,v in d.get('extras',{}).items()}, round(d['e2e']['value']/1e9,2) if d.get('e2e') else None)
"; done
