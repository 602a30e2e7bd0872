cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python tools/bench_grad.py > gpurun_out/grad_fast.log 2>&1; echo "rc=$?" >> gpurun_out/grad_fast.log
timeout 300 python tools/debug_normals.py > gpurun_out/debug_normals.log 2>&1; echo "rc=$?" >> gpurun_out/debug_normals.log
timeout 900 python -m pytest tests/test_gpu_objectives.py -x -q -p no:cacheprovider > gpurun_out/pytest_obj.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_obj.log
