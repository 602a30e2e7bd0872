# single-GPU pass of the final session (same steps as tools/gpu_final1.sh) -> gpurun_out/r3_final
# single-GPU round-end pass: tests, smoke, default bench + reference arm, profiles
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r3_final
O=gpurun_out/r3_final
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total,power.limit --format=csv > $O/nvsmi.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_ref.log 2>&1; echo "rc=$?" >> $O/bench_ref.log
timeout 600 python bench.py > $O/bench_default.log 2>&1; echo "rc=$?" >> $O/bench_default.log
timeout 600 python bench.py --steps 50 --warmup 5 --no-cpu --no-e2e --strategy d1d > $O/bench_d1d.log 2>&1
timeout 600 python bench.py --steps 50 --warmup 5 --no-cpu --no-e2e --strategy adpsgd_fixed > $O/bench_ad.log 2>&1
timeout 300 python bench.py --steps 200 --warmup 5 --learners 16 --dim 1048576 --no-cpu --no-e2e > $O/bench_c1.log 2>&1
timeout 600 python bench.py --steps 20 --warmup 3 --learners 128 --dim 43154944 --no-cpu --no-e2e > $O/bench_c3.log 2>&1
# launch list of the default bench command (cold, serialised; shares only)
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_default.csv python bench.py --steps 2 --warmup 3 --cpu-seconds 1 > $O/ncu_launches.log 2>&1
# full captures of the dominant kernels
timeout 900 ncu --set full --clock-control none --import-source on -k regex:mix_tma -s 3 -c 1 -o $O/prof_c2_rad python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e > $O/ncu_c2.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:mix_tma -s 3 -c 1 -o $O/prof_c4_d1d python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e --strategy d1d > $O/ncu_c4.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:mix_tma -s 3 -c 1 -o $O/prof_c2_rad_bf16 python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e --dtype bfloat16 > $O/ncu_c2bf.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__issue_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:zig_ --csv --log-file $O/launches_normals_c2.csv python tools/grad_once.py 64 25557032 > $O/ncu_zig.log 2>&1
timeout 600 python tools/bench_training.py > $O/bench_training.log 2>&1
timeout 300 python tools/bench_trace.py > $O/bench_trace.log 2>&1
timeout 300 python tools/bench_grad.py > $O/bench_grad.log 2>&1
timeout 300 python tools/d1d_step_probe.py > $O/d1d_step.json 2>&1
timeout 900 python -m pytest tests/test_gpu_reference_suite.py -q -p no:cacheprovider > $O/pytest_refsuite.log 2>&1
echo done > $O/done.txt
