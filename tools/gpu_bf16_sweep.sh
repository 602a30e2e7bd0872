# bf16 ring-tile sweep at C2: CTA shape (RINGMIX_RING_NT) x stage size (RINGMIX_STAGE_KB)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
: > gpurun_out/bf16_sweep.log
for NT in 512 256; do for KB in 0 24 32 48 64; do
 if [ $KB = 0 ]; then unset RINGMIX_STAGE_KB; else export RINGMIX_STAGE_KB=$KB; fi
 RINGMIX_RING_NT=$NT timeout 300 python bench.py --steps 50 --warmup 5 --dtype bfloat16 --no-cpu --no-e2e 2>&1 | grep -o '"frac": [0-9.]*\|"ms_per_step": [0-9.]*' | tr '\n' ' ' | sed "s/^/NT=$NT KB=$KB /" >> gpurun_out/bf16_sweep.log; echo >> gpurun_out/bf16_sweep.log
done; done
