cd $GRAFT_REPO_ROOT
O=gpurun_out/r2g; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_simulation.py -q -x > $O/pytest_sim.log 2>&1; echo rc=$? >> $O/pytest_sim.log
timeout 300 python bench.py --learners 16 --dim 1048576 --no-cpu --no-e2e --steps 400 > $O/bench_c1_graph.log 2>&1
for dt in float32 bfloat16 float64; do timeout 300 python tools/probe_mix.py --mode mean --dtype $dt --n 20 > $O/d1d_$dt.jsonl 2>&1; done
timeout 300 python tools/probe_mix.py --dtype float64 --n 20 > $O/rad_float64.jsonl 2>&1
tail -3 $O/*
