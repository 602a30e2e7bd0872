# 2-GPU pass (round 2): multi-GPU tests (dist_check incl. peer-table forms), NVLink counter
# probe, bench.py self-launch at N=2 (position layout on C3 + extras), D1D, and N=1.
cd $GRAFT_REPO_ROOT
O=gpurun_out/n2_r2; mkdir -p $O
nvidia-smi topo -m > $O/topo.txt 2>&1
timeout 300 python tools/probe_nvlink_counters.py > $O/nvlink_probe.log 2>&1
timeout 900 python -m pytest tests/test_gpu_multi.py tests/test_gpu_integration.py -x -q > $O/pytest_multi.log 2>&1; echo "rc=$?" >> $O/pytest_multi.log
timeout 900 python bench.py --gpus 2 > $O/bench_n2.log 2>&1; echo "rc=$?" >> $O/bench_n2.log
timeout 600 python bench.py --gpus 2 --strategy d1d --no-extras > $O/bench_n2_d1d.log 2>&1; echo "rc=$?" >> $O/bench_n2_d1d.log
timeout 900 python bench.py > $O/bench_n1.log 2>&1; echo "rc=$?" >> $O/bench_n1.log
timeout 300 python bench.py --impl reference --gpus 2 --steps 5 --warmup 3 > $O/ref_n2.log 2>&1
tail -3 $O/*.log
