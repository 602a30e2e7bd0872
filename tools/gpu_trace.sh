cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_objectives.py tests/test_gpu_simulation.py -q -p no:cacheprovider > gpurun_out/pytest_trace.log 2>&1; echo rc=$? >> gpurun_out/pytest_trace.log
timeout 600 python tools/bench_training.py > gpurun_out/bench_training.log 2>&1
timeout 600 python tools/prof_training.py > gpurun_out/prof_training.log 2>&1
