cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
: > gpurun_out/zspec_sweep.log
for m in 1 8 10 12; do
  touch paper_2002_01119_b200/csrc/normal.cu
  make -C paper_2002_01119_b200/csrc NVFLAGS="-O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr -DRM_ZSPEC_MINB=$m" > /dev/null 2>&1 || echo "build fail $m" >> gpurun_out/zspec_sweep.log
  TAG=minb$m timeout 300 python tools/grad_once.py 64 25557032 >> gpurun_out/zspec_sweep.log 2>&1
done
