cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
export RINGMIX_TILE_COLS=128
timeout 600 python bench.py --steps 10 --warmup 3 --strategy d1d --no-cpu --no-e2e > gpurun_out/bench_c4_scalar.log 2>&1
unset RINGMIX_TILE_COLS
CMD="python tools/bench_grad.py"
timeout 300 $CMD > gpurun_out/plain_grad.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:zig_ -s 12 -c 6 -o gpurun_out/prof_zig $CMD > gpurun_out/ncu_zig.log 2>&1
