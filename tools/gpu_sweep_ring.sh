cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
SW_KB=0,48,80,96 timeout 300 python tools/sweep_ring.py > gpurun_out/sweep_ring.log 2>&1
RINGMIX_RING_NT=256 SW_KB=24,32,48 timeout 300 python tools/sweep_ring.py >> gpurun_out/sweep_ring.log 2>&1
SW_L=16 SW_D=16777216 SW_KB=0,32 timeout 300 python tools/sweep_ring.py >> gpurun_out/sweep_ring.log 2>&1
SW_L=16 SW_D=16777216 RINGMIX_RING_NT=256 SW_KB=24,32 timeout 300 python tools/sweep_ring.py >> gpurun_out/sweep_ring.log 2>&1
SW_L=128 SW_D=10788736 SW_KB=0,96 timeout 300 python tools/sweep_ring.py >> gpurun_out/sweep_ring.log 2>&1
SW_L=128 SW_D=10788736 RINGMIX_RING_NT=256 SW_KB=32,48 timeout 300 python tools/sweep_ring.py >> gpurun_out/sweep_ring.log 2>&1
