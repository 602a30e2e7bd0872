cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_mix.py tests/test_gpu_simulation.py tests/test_gpu_objectives.py tests/test_gpu_shard.py -x -q -p no:cacheprovider > gpurun_out/pytest_mean.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_mean.log
: > gpurun_out/mean_bench.log
for st in d1d rand_psgd; do for dt in float32 bfloat16 float64; do
timeout 300 python bench.py --steps 20 --warmup 3 --strategy $st --dtype $dt --no-cpu --no-e2e 2>&1 | grep -o '"frac": [0-9.]*\|"ms_per_step": [0-9.]*' | tr '\n' ' ' | sed "s/^/$st $dt /" >> gpurun_out/mean_bench.log; echo >> gpurun_out/mean_bench.log
done; done
