set -x
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python tools/sweep_tile.py > gpurun_out/sweep1.log 2>&1
CMD="python bench.py --steps 4 --warmup 3 --no-cpu --no-e2e"
timeout 300 $CMD > gpurun_out/plain_c2.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:mix_tma -s 3 -c 1 -o gpurun_out/prof_c2 $CMD > gpurun_out/ncu_c2.log 2>&1
CMD1="python bench.py --steps 4 --warmup 3 --no-cpu --no-e2e --learners 16 --dim 1048576"
timeout 300 $CMD1 > gpurun_out/plain_c1.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:mix_tma -s 3 -c 1 -o gpurun_out/prof_c1 $CMD1 > gpurun_out/ncu_c1.log 2>&1
ls -la gpurun_out
