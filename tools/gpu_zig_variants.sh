
# A/B timing of generator build variants (paper_2002_01119_b200/lib/variants/*.so): C2 gradient time + bit-identity tests
L=paper_2002_01119_b200/lib
mkdir -p gpurun_out/zv
for v in ${VARIANTS:-orig k0 k1 k2}; do
  cp $L/variants/libringmix_b200_$v.so $L/libringmix_b200.so
  timeout 300 python -c "
import sys; sys.path.insert(0,'tools'); import bench_grad as b
b.main(64, 25_557_032, reps=9); b.compare_paths(64, 25_557_032)" > gpurun_out/zv/$v.log 2>&1
  if [ $v != orig ]; then timeout 600 python -m pytest tests -q -x -m gpu -k "objectives or normal or grad" >> gpurun_out/zv/$v.log 2>&1; echo rc=$? >> gpurun_out/zv/$v.log; fi
done
