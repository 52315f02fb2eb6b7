#!/bin/bash
# Builds libixb.so with extra nvcc defines into scratch_libs/<name>/ (perf
# experiments; load with IXB_LIB_PATH=scratch_libs/<name>/libixb.so).
# usage: tools/build_variant.sh <name> <source.cu> -DMACRO ...
set -e
name=$1; src=$2; shift 2
root=$(cd "$(dirname "$0")/.." && pwd)
out=$root/scratch_libs/$name
mkdir -p "$out/build"
cd "$root/paper_2510_17505_b200/csrc"
make -s -j8 >/dev/null
for o in ../build/*.o; do cp "$o" "$out/build/"; done
obj=$out/build/$(basename "${src%.cu}").o
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a "$@" -O3 -lineinfo -std=c++17 \
  -Xcompiler -fPIC --expt-relaxed-constexpr -c "$src" -o "$obj"
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o "$out/libixb.so" \
  "$out"/build/*.o -lcudart_static -ldl -lpthread -lrt
echo "$out/libixb.so"
