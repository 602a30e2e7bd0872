# A/B: exact u52 -> double by the 2^52 bias (default build) vs I2F (variant i2f)
cd $GRAFT_REPO_ROOT
O=gpurun_out/zig_i2f; mkdir -p $O
L=paper_2002_01119_b200/lib
cp $L/libringmix_b200.so $L/libringmix_b200.so.orig
for rep in 1 2; do
  for v in orig i2f; do
    if [ $v = orig ]; then cp $L/libringmix_b200.so.orig $L/libringmix_b200.so; else cp $L/variants/libringmix_b200_$v.so $L/libringmix_b200.so; fi
    timeout 300 python -c "
import sys; sys.path.insert(0,'tools'); import bench_grad as b
b.main(64, 25_557_032, reps=7)" > $O/grad_${v}_$rep.log 2>&1
  done
done
cp $L/libringmix_b200.so.orig $L/libringmix_b200.so
timeout 900 python -m pytest tests/test_gpu_objectives.py -q -x > $O/pytest_obj.log 2>&1; echo rc=$? >> $O/pytest_obj.log
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv python -c "
import sys; sys.path.insert(0,'tools'); import bench_grad as b
b.main(64, 25_557_032, reps=1)" > $O/launches.csv 2>&1
tail -2 $O/*.log
