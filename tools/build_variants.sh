#!/bin/bash
# Kernel tuning: build libqtng variants, one per "tag:-DFLAGS ..." argument,
# into build/variants/libqtng_<tag>.so (host objects from the last `make`).
set -e
cd "$(dirname "$0")/../paper_2204_06045_b200/csrc"
mkdir -p ../../build/variants
rm -f ../../build/variants/*.so
for v in "$@"; do
  tag=${v%%:*}; flags=${v#*:}
  nvcc -std=c++17 -O3 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC -Xptxas -v \
       -I../../include $flags -c kernels.cu -o ../../build/variants/k_$tag.o 2> ../../build/variants/ptxas_$tag.txt
  nvcc -std=c++17 -O3 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC \
       -I../../include $flags -DQTNG_C64=1 -c kernels.cu -o ../../build/variants/k64_$tag.o
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -o ../../build/variants/libqtng_$tag.so \
       ../../build/obj/host.o ../../build/obj/walk.o ../../build/obj/plan.o ../../build/obj/capi.o \
       ../../build/obj/sv.o ../../build/obj/peak.o ../../build/variants/k_$tag.o ../../build/variants/k64_$tag.o -lpthread
  echo "$tag: $(grep -A2 seg_kernel ../../build/variants/ptxas_$tag.txt | grep -E 'registers|spill' | tr '\n' ' ' | tr -s ' ')"
done
