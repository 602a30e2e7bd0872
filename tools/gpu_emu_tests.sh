mkdir -p gpurun_out/emu
timeout 900 python -m pytest tests/test_gpu_emulated_world.py tests/test_gpu_fullsize.py -x -q -v > gpurun_out/emu/pytest_new.log 2>&1; echo "rc=$?" >> gpurun_out/emu/pytest_new.log
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/emu/pytest_all.log 2>&1; echo "rc=$?" >> gpurun_out/emu/pytest_all.log
tail -30 gpurun_out/emu/pytest_new.log; tail -5 gpurun_out/emu/pytest_all.log
