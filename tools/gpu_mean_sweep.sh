# D1D (mean tiles) stage-size sweep at C4 per storage type
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
: > gpurun_out/mean_sweep.log
for dt in float32 bfloat16 float64; do for KB in 0 16 24; do
 if [ $KB = 0 ]; then unset RINGMIX_STAGE_KB; else export RINGMIX_STAGE_KB=$KB; fi
 timeout 300 python bench.py --steps 50 --warmup 5 --strategy d1d --dtype $dt --no-cpu --no-e2e 2>&1 | grep -o '"frac": [0-9.]*\|"ms_per_step": [0-9.]*' | tr '\n' ' ' | sed "s/^/$dt KB=$KB /" >> gpurun_out/mean_sweep.log; echo >> gpurun_out/mean_sweep.log
done; done
