cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
: > gpurun_out/sweep_ring.log
for rep in 1 2 3; do
SW_KB=48,64,32,48,64 timeout 300 python tools/sweep_ring.py >> gpurun_out/sweep_ring.log 2>&1
SW_L=16 SW_D=16777216 SW_KB=64,32,16,32 timeout 300 python tools/sweep_ring.py >> gpurun_out/sweep_ring.log 2>&1
SW_L=16 SW_D=16777216 RINGMIX_RING_NT=256 SW_KB=24,16,32 timeout 300 python tools/sweep_ring.py >> gpurun_out/sweep_ring.log 2>&1
SW_L=16 SW_D=1048576 SW_KB=64,32,16 timeout 300 python tools/sweep_ring.py >> gpurun_out/sweep_ring.log 2>&1
SW_L=16 SW_D=1048576 RINGMIX_RING_NT=256 SW_KB=24,16 timeout 300 python tools/sweep_ring.py >> gpurun_out/sweep_ring.log 2>&1
done
