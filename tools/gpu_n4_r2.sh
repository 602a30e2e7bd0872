# 4-GPU pass (round 2): the driver's scaling commands (both arms, N = 1, 2, 4), the
# multi-GPU tests on 4 GPUs, D1D at N = 4, and a sanitizer-free dist_check at n = 3 (ragged).
cd $GRAFT_REPO_ROOT
O=gpurun_out/n4_r2; mkdir -p $O
nvidia-smi topo -m > $O/topo.txt 2>&1
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
( time timeout 900 python bench.py ) > $O/drv_ours_n1.log 2>&1
( time timeout 600 python bench.py --impl reference ) > $O/drv_ref_n1.log 2>&1
for n in 2 4; do
  ( time timeout 900 $TR --nproc-per-node $n --master-port $((29800+n)) bench.py --gpus $n ) > $O/drv_ours_n$n.log 2>&1
  ( time timeout 600 $TR --nproc-per-node $n --master-port $((29810+n)) bench.py --impl reference --gpus $n --steps 5 --warmup 3 ) > $O/drv_ref_n$n.log 2>&1
done
( time timeout 600 python bench.py --gpus 4 --strategy d1d --no-extras ) > $O/d1d_n4.log 2>&1
( time timeout 600 python bench.py --gpus 4 --strategy adpsgd_fixed --no-extras ) > $O/adpsgd_n4.log 2>&1
timeout 900 python -m pytest tests/test_gpu_multi.py tests/test_gpu_integration.py -x -q > $O/pytest_multi.log 2>&1; echo "rc=$?" >> $O/pytest_multi.log
CHK_L=10 CHK_D=4099 timeout 600 $TR --nproc-per-node 3 --master-port 29831 tools/dist_check.py > $O/dist_check_n3.log 2>&1; echo "rc=$?" >> $O/dist_check_n3.log
tail -2 $O/*.log
