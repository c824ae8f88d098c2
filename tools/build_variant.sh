#!/bin/bash
# Build libdarm_gpu.so variants with extra -D flags into variants/<name>/ (load
# one with DARM_GPU_LIB=variants/<name>/libdarm_gpu.so).  Usage:
#   tools/build_variant.sh <name> -DFOO=1 ...
set -e
name=$1; shift
out=variants/$name
mkdir -p $out/obj
src=paper_2107_05681_b200/csrc
FL="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O2 -Iinclude --expt-relaxed-constexpr"
pids=()
for f in $src/*.cu; do
  b=$(basename $f .cu); extra=""
  [ $b = srad ] && extra="-fmad=false"
  nvcc $FL $extra "$@" -c -o $out/obj/$b.o $f & pids+=($!)
done
for p in "${pids[@]}"; do wait $p; done
nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o $out/libdarm_gpu.so $out/obj/*.o -Xlinker --no-undefined -lpthread
rm -rf $out/obj
echo built $out/libdarm_gpu.so
