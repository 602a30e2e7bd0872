cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 300 python tools/bench_d1d_kernels.py > gpurun_out/d1dk.log 2>&1 && \
timeout 600 ncu --set full --clock-control none -k regex:apply_mean -s 3 -c 1 -o gpurun_out/prof_apply python tools/bench_d1d_kernels.py > gpurun_out/ncu_apply.log 2>&1
