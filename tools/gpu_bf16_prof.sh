cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python bench.py --steps 3 --warmup 3 --dtype bfloat16 --no-cpu --no-e2e > /dev/null 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:mix_tma -c 1 -o gpurun_out/prof_rad_bf16 python bench.py --steps 3 --warmup 3 --dtype bfloat16 --no-cpu --no-e2e > gpurun_out/ncu_rad_bf16.log 2>&1
