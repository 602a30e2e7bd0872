cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
for rep in 1 2; do
timeout 300 python bench.py --steps 400 --warmup 10 --learners 16 --dim 1048576 --no-cpu --no-e2e > gpurun_out/cfg_c1_$rep.log 2>&1
timeout 300 python bench.py --steps 100 --warmup 5 --learners 16 --dim 16777216 --no-cpu --no-e2e > gpurun_out/cfg_c1big_$rep.log 2>&1
timeout 300 python bench.py --steps 100 --warmup 5 --no-cpu --no-e2e > gpurun_out/cfg_c2_$rep.log 2>&1
done
