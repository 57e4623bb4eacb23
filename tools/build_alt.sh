#!/bin/bash
# Build the current csrc/ into tools/alt/$1.so (for A/B timing with tools/ab_i8.py).
set -e
name=$1
d=$(mktemp -d)
cd "$(dirname "$0")/../paper_1304_2272_b200/csrc"
for f in *.cu; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Xcompiler -fPIC \
    --expt-relaxed-constexpr $GG_ALT_FLAGS -c "$f" -o "$d/${f%.cu}.o" &
done
wait
mkdir -p ../../tools/alt
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o "../../tools/alt/$name.so" "$d"/*.o \
  -lcudart_static -lrt -lpthread -ldl
rm -rf "$d"
echo "built tools/alt/$name.so"
