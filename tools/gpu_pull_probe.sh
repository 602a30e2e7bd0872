cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python tools/pull_probe.py > gpurun_out/pull_probe.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:mix_shard -s 4 -c 1 -o gpurun_out/prof_pull python tools/pull_probe.py > gpurun_out/ncu_pull.log 2>&1
echo rc=$? >> gpurun_out/pull_probe.log
