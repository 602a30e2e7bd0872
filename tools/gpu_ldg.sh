cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_mix.py tests/test_gpu_simulation.py -x -q -p no:cacheprovider > gpurun_out/pytest_mix.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_mix.log
: > gpurun_out/ldg.log
for rep in 1 2 3; do
for G in ldg stage; do
RINGMIX_RING_G=$G SW_KB=0 timeout 300 python tools/sweep_ring.py | sed "s/^/$G /" >> gpurun_out/ldg.log 2>&1
RINGMIX_RING_G=$G SW_L=128 SW_D=10788736 SW_KB=0 timeout 300 python tools/sweep_ring.py | sed "s/^/$G /" >> gpurun_out/ldg.log 2>&1
done; done
