cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python tools/grad_once.py 64 25557032 > gpurun_out/grad_once.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:zig_ --csv --log-file gpurun_out/zig_launches.csv python tools/grad_once.py 64 25557032 > gpurun_out/ncu_zl.log 2>&1
echo rc=$? >> gpurun_out/grad_once.log
