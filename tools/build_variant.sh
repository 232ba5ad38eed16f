#!/bin/bash
# Build a variant of the C-ABI library with extra preprocessor flags, for
# tools/ab.py: tools/build_variant.sh build/lib_x.so -DLSQ_SELF_FEED=0
set -e
out=$1; shift
tag=$(basename "$out" .so)
dir=build/varobj/$tag
mkdir -p "$dir"
objs=()
for f in paper_1512_08017_b200/csrc/*.cu; do
  o=$dir/$(basename "$f" .cu).o
  /usr/local/cuda/bin/nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo --fmad=false \
    -Xcompiler -fPIC -Iinclude "$@" -c -o "$o" "$f" &
  objs+=("$o")
done
wait
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o "$out" "${objs[@]}" -lcudart
