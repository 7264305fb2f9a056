#!/bin/bash
# Build libdetseries_b200.so with implementation-variant macros into
# build_variants/<name>/ (A/B timing on the GPU: DS_LIB_PATH=<that .so>).
# usage: tools/build_variant.sh NAME "-DDS_VAR_MMAWARP=0 -DDS_VAR_MULSHIFT=0 ..."
set -e
name=$1; flags=$2
ROOT=$(cd "$(dirname "$0")/.." && pwd)
out=$ROOT/build_variants/$name
mkdir -p "$out"
cd "$ROOT/paper_1308_1536_b200/csrc"
NV="/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr $flags"
for f in ds_engine ds_update ds_tc ds_gen; do $NV -c -o "$out/$f.o" $f.cu & done; wait
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -cudart static -shared -o "$out/libdetseries_b200.so" "$out"/*.o
rm -f "$out"/*.o
echo "$out/libdetseries_b200.so"
