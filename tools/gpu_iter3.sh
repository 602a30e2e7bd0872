cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for cw in 0 64 128; do
  if [ $cw -gt 0 ]; then export RINGMIX_TILE_COLS=$cw; else unset RINGMIX_TILE_COLS; fi
  timeout 300 python bench.py --steps 50 --warmup 5 --strategy d1d --no-cpu --no-e2e > gpurun_out/bench_c4_cw$cw.log 2>&1
done
unset RINGMIX_TILE_COLS
CMD="python bench.py --steps 4 --warmup 3 --no-cpu --no-e2e --strategy d1d"
timeout 300 $CMD > gpurun_out/plain_d1d.log 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:mix_tma -s 3 -c 1 -o gpurun_out/prof_d1d $CMD > gpurun_out/ncu_d1d.log 2>&1
