cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python tools/bench_grad.py > gpurun_out/bench_grad.log 2>&1; echo "rc=$?" >> gpurun_out/bench_grad.log
timeout 300 python bench.py --steps 400 --warmup 10 --learners 16 --dim 1048576 --no-cpu --no-e2e > gpurun_out/bench_c1.log 2>&1
timeout 300 python bench.py --steps 50 --warmup 5 --learners 128 --dim 43154944 --no-cpu --no-e2e > gpurun_out/bench_c3.log 2>&1
timeout 300 python bench.py --steps 50 --warmup 5 --strategy d1d --no-cpu --no-e2e > gpurun_out/bench_c4.log 2>&1
timeout 300 python bench.py --steps 50 --warmup 5 --strategy adpsgd_fixed --no-cpu --no-e2e > gpurun_out/bench_ad.log 2>&1
timeout 300 python bench.py --steps 50 --warmup 5 --dtype bfloat16 --no-cpu --no-e2e > gpurun_out/bench_bf16.log 2>&1
timeout 300 python bench.py --steps 30 --warmup 5 --dtype float64 --no-cpu --no-e2e > gpurun_out/bench_f64.log 2>&1
