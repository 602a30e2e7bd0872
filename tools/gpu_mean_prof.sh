cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for v in "bfloat16 1" "float32 1"; do set -- $v
RINGMIX_MEAN_STAGE_G=$2 timeout 300 python bench.py --steps 3 --warmup 3 --strategy d1d --dtype $1 --no-cpu --no-e2e > /dev/null 2>&1 && \
RINGMIX_MEAN_STAGE_G=$2 timeout 600 ncu --set full --clock-control none --import-source on -k regex:mix_tma -c 1 -o gpurun_out/prof_mean_$1_sg$2 python bench.py --steps 3 --warmup 3 --strategy d1d --dtype $1 --no-cpu --no-e2e > gpurun_out/ncu_mean_$1_$2.log 2>&1
done
