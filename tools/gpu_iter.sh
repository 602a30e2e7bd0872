# quick iteration: gpu tests + tile sweep + short bench + ncu of the C2 kernel
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python tools/sweep_tile.py > gpurun_out/sweep.log 2>&1
timeout 600 python bench.py --steps 100 --warmup 5 --cpu-seconds 3 > gpurun_out/bench_c2.log 2>&1; echo "rc=$?" >> gpurun_out/bench_c2.log
CMD="python bench.py --steps 4 --warmup 3 --no-cpu --no-e2e"
timeout 300 $CMD > gpurun_out/plain_c2.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:mix_tma -s 3 -c 1 -o gpurun_out/prof_c2_v3 $CMD > gpurun_out/ncu_c2.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv $CMD > gpurun_out/ncu_launches.log 2>&1
