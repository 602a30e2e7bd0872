# what the driver does at round end (N=1 and the scaling run), both arms
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
( time timeout 900 python bench.py ) > gpurun_out/drv_ours_n1.log 2>&1
( time timeout 900 python bench.py --impl reference ) > gpurun_out/drv_ref_n1.log 2>&1
for n in 2 4; do
  [ $n -gt $N ] && continue
  ( time timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29800+n)) bench.py --gpus $n ) > gpurun_out/drv_ours_n$n.log 2>&1
  ( time timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29810+n)) bench.py --impl reference --gpus $n --steps 5 --warmup 3 ) > gpurun_out/drv_ref_n$n.log 2>&1
done
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
