# single GPU: warp-specialised trace kernel (tests, timing, ncu), compute-sanitizer pass,
# full pytest -m gpu.
cd $GRAFT_REPO_ROOT
O=gpurun_out/r2c; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_objectives.py -q -x > $O/pytest_objectives.log 2>&1; echo rc=$? >> $O/pytest_objectives.log
timeout 300 python tools/bench_trace.py > $O/bench_trace_ws.log 2>&1
RINGMIX_TRACE_IMPL=barrier timeout 300 python tools/bench_trace.py > $O/bench_trace_barrier.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:trace_ws -s 2 -c 1 -o $O/trace_ws_c2 python tools/bench_trace.py > $O/ncu_trace.log 2>&1
timeout 2400 bash tools/sanitize.sh > $O/sanitize.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.log 2>&1; echo rc=$? >> $O/pytest_gpu.log
tail -3 $O/*.log
