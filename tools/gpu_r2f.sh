cd $GRAFT_REPO_ROOT
O=gpurun_out/r2f; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_objectives.py tests/test_gpu_harness.py -q -x > $O/pytest_trace.log 2>&1; echo rc=$? >> $O/pytest_trace.log
timeout 300 python tools/bench_trace.py > $O/bench_trace.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:trace_stats_tma -s 2 -c 1 -o $O/trace_c2 python tools/bench_trace.py > $O/ncu_trace.log 2>&1
tail -3 $O/*.log
