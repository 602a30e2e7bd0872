#!/bin/bash
# trace_stats: tests + C2 timing (+ ncu launch time of the tiled kernel)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
o=gpurun_out/${1:-trace_ab}; mkdir -p $o
timeout 900 python -m pytest tests/test_gpu_objectives.py -x -q -k trace 2>&1 | tail -2 > $o/tests.log
timeout 600 python tools/bench_trace.py > $o/bench.json 2> $o/bench.err
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none --csv -k regex:trace_stats_tma \
  --log-file $o/launches.csv python tools/bench_trace.py > $o/ncu.log 2>&1
cat $o/tests.log $o/bench.json
