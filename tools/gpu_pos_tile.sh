# position layout: tile width sweep (remote store segment length)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --nproc-per-node $N"
: > gpurun_out/pos_tile.log
for CW in 0 256 64; do
 if [ $CW = 0 ]; then unset RINGMIX_TILE_COLS; else export RINGMIX_TILE_COLS=$CW; fi
 timeout 300 $TR --master-port 29931 bench.py --gpus $N --steps 30 --warmup 5 --no-cpu --no-e2e --layout position 2>&1 | grep -o '"ms_per_step": [0-9.]*' | sed "s/^/cw=$CW /" >> gpurun_out/pos_tile.log
done
