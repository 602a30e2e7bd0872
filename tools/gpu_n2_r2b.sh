# 2-GPU pass b: NVML / ncu NVLink counters, the single-process layout harness under ncu,
# bench.py --gpus 2 (position layout on C3 + extras) and D1D.
cd $GRAFT_REPO_ROOT
O=gpurun_out/n2_r2b; mkdir -p $O
timeout 300 python tools/probe_nvlink_counters.py > $O/nvlink_probe.log 2>&1
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,nvlrx__bytes.sum,nvltx__bytes.sum,nvlrx__bytes_data_user.sum,nvltx__bytes_data_user.sum
for lay in position learner; do
  PP_LAYOUT=$lay timeout 300 python tools/pos_probe.py > $O/probe_$lay.log 2>&1
  PP_LAYOUT=$lay PP_STEPS=6 timeout 600 ncu --metrics $M --clock-control none -k regex:mix_shard -s 3 -c 2 --csv python tools/pos_probe.py > $O/ncu_$lay.csv 2> $O/ncu_$lay.err
done
timeout 900 python bench.py --gpus 2 > $O/bench_n2.log 2>&1; echo "rc=$?" >> $O/bench_n2.log
timeout 600 python bench.py --gpus 2 --strategy d1d --no-extras > $O/bench_n2_d1d.log 2>&1; echo "rc=$?" >> $O/bench_n2_d1d.log
tail -3 $O/*.log
