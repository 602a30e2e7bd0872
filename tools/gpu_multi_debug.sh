# learner-sharded RAD bit-identity at ragged shard sizes, per layout / rank / step, repeated
cd $GRAFT_REPO_ROOT
O=gpurun_out/multi_debug; mkdir -p $O
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
for rep in 1 2 3; do
for n in 3 4; do
  for LD in "8 4099" "5 4099" "67 100003" "13 20011"; do
    set -- $LD
    echo "n=$n L=$1 d=$2 rep=$rep" >> $O/out.txt
    CHK_L=$1 CHK_D=$2 timeout 300 $TR --nproc-per-node $n --master-port $((29600+n)) tools/dist_check.py 2>>$O/err.txt | grep '^{' >> $O/out.txt
  done
done
done
timeout 900 python -m pytest tests/test_gpu_multi.py tests/test_gpu_shard.py -q -p no:cacheprovider > $O/pytest_multi.log 2>&1; echo "rc=$?" >> $O/pytest_multi.log
