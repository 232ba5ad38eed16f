#!/bin/bash
# Build a variant of the C-ABI library that differs only in
# k_power_sums.cu's preprocessor flags (every other object from build/obj,
# so `make` must have run): tools/build_ps_variant.sh build/lib_x.so -DLSQ_PRODUCT_MIN=13
set -e
out=$1; shift
tag=$(basename "$out" .so)
mkdir -p build/varobj/$tag
/usr/local/cuda/bin/nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo --fmad=false \
  -Xcompiler -fPIC -Iinclude "$@" -c -o build/varobj/$tag/k_power_sums.o paper_1512_08017_b200/csrc/k_power_sums.cu
objs=$(ls build/obj/*.o | grep -v k_power_sums.o)
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o "$out" $objs build/varobj/$tag/k_power_sums.o -lcudart
