#!/bin/bash
# Build a variant of the C-ABI library that differs only in one translation
# unit's preprocessor flags (every other object from build/obj, so `make`
# must have run): tools/build_tu_variant.sh k_batched build/lib_x.so -DMACRO=1
set -e
tu=$1; out=$2; shift 2
tag=$(basename "$out" .so)
mkdir -p build/varobj/$tag
/usr/local/cuda/bin/nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo --fmad=false \
  -Xcompiler -fPIC -Iinclude "$@" -c -o build/varobj/$tag/$tu.o paper_1512_08017_b200/csrc/$tu.cu
objs=$(ls build/obj/*.o | grep -v "/$tu.o")
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o "$out" $objs build/varobj/$tag/$tu.o -lcudart
