cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r3_mixncu
cp paper_2002_01119_b200/lib/libringmix_b200.so /tmp/main.so
VARIANTS="orig k3 orig k3" bash tools/gpu_zig_variants.sh
cp /tmp/main.so paper_2002_01119_b200/lib/libringmix_b200.so
grep -h "grad_ms\|passed\|failed\|rc=" gpurun_out/zv/*.log
python -m pytest tests/test_gpu_emulated_world.py -q -x -p no:cacheprovider -k "placed or placement" > gpurun_out/r3_mixncu/emu.log 2>&1; tail -2 gpurun_out/r3_mixncu/emu.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:mix_tma -s 3 -c 1 -o gpurun_out/r3_mixncu/c2_rad python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/r3_mixncu/ncu.log 2>&1; tail -2 gpurun_out/r3_mixncu/ncu.log
