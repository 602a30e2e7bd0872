cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python tools/grad_once.py 64 25557032 > gpurun_out/zprof.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:zig_spec -c 1 -o gpurun_out/prof_zspec_c2 python tools/grad_once.py 64 25557032 >> gpurun_out/zprof.log 2>&1
echo rc=$? >> gpurun_out/zprof.log
