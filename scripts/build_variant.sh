#!/bin/sh
# Build a variant of libcotten.so into build_variants/lib_<name>.so with extra nvcc flags.
#   scripts/build_variant.sh trace -DCOTTEN_TC_TRACE=1
set -e
cd "$(dirname "$0")/.."
name=$1; shift
mkdir -p build_variants/obj_$name
NV="/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC $*"
$NV -c -o build_variants/obj_$name/capi.o paper_2602_06935_b200/csrc/cotten_capi.cu
$NV -c -o build_variants/obj_$name/enc.o paper_2602_06935_b200/csrc/encoder.cu
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o build_variants/lib_$name.so build_variants/obj_$name/capi.o build_variants/obj_$name/enc.o -lcublas
echo built build_variants/lib_$name.so
