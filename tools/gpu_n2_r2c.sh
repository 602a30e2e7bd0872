# 2-GPU pass c: placed ring-position layout (tests, dist_check, bench placed vs fixed)
cd $GRAFT_REPO_ROOT
O=gpurun_out/n2_r2c; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_emulated_world.py -q -x > $O/pytest_emu.log 2>&1; echo rc=$? >> $O/pytest_emu.log
timeout 900 python -m pytest tests/test_gpu_multi.py -q -x > $O/pytest_multi.log 2>&1; echo rc=$? >> $O/pytest_multi.log
timeout 900 python bench.py --gpus 2 --no-extras > $O/bench_n2_placed.log 2>&1; echo rc=$? >> $O/bench_n2_placed.log
RINGMIX_POS_PLACEMENT=fixed timeout 900 python bench.py --gpus 2 --no-extras --no-e2e > $O/bench_n2_fixed.log 2>&1; echo rc=$? >> $O/bench_n2_fixed.log
tail -3 $O/*.log | cut -c1-400
