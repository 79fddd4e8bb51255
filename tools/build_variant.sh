#!/bin/bash
# Build an A/B variant of libfftmv_cuda.so with extra nvcc flags into
# build/alt/<name>/libfftmv_cuda.so (load it with FMV_LIB_PATH=...).
#   tools/build_variant.sh block416 -DFMV_BLOCK_CONS=416
set -e
cd "$(dirname "$0")/.."
name=$1; shift
out=build/alt/$name
mkdir -p $out
objs=()
for f in paper_2508_10202_b200/csrc/*.cu; do
  b=$(basename $f .cu)
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++20 -Xcompiler -fPIC \
    --expt-relaxed-constexpr "$@" -c -o $out/$b.o $f &
  objs+=($out/$b.o)
done
for f in paper_2508_10202_b200/csrc/*.cpp; do
  b=$(basename $f .cpp)
  g++ -std=c++20 -O2 -fPIC -c -o $out/$b.o $f &
  objs+=($out/$b.o)
done
wait
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $out/libfftmv_cuda.so "${objs[@]}" -ldl -lcudart -lpthread
echo $out/libfftmv_cuda.so
