#!/bin/bash
# Build a variant of the product library with extra nvcc flags into
# paper_2002_01119_b200/lib/variants/libringmix_b200_<name>.so (A/B timing on the GPU box).
# usage: tools/build_variant.sh <name> "<extra nvcc flags>"
set -e
cd "$(dirname "$0")/../paper_2002_01119_b200/csrc"
name=$1; shift
B=../../build/variant_$name
mkdir -p $B ../lib/variants
for f in abi perm mix dl host shard normal trace; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
    --expt-relaxed-constexpr $* -c $f.cu -o $B/$f.o &
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o ../lib/variants/libringmix_b200_$name.so \
  $B/*.o -lcudart_static -lrt -ldl -lpthread
echo built ../lib/variants/libringmix_b200_$name.so
