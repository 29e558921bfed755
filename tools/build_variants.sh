#!/bin/bash
# Kernel tuning: build libqtng variants with different occupancy bounds.
set -e
cd "$(dirname "$0")/../paper_2204_06045_b200/csrc"
mkdir -p ../../build/variants
CU=/usr/local/cuda
for v in "3 3" "4 3" "4 4" "3 2" "2 2"; do
  set -- $v
  tag=t2_$1_t4_$2
  nvcc -std=c++17 -O3 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC -Xptxas -v \
       -I../../include -DQTNG_MINB_T2=$1 -DQTNG_MINB_T4=$2 -c kernels.cu -o ../../build/variants/k_$tag.o 2> ../../build/variants/ptxas_$tag.txt
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -o ../../build/variants/libqtng_$tag.so \
       ../../build/obj/host.o ../../build/obj/plan.o ../../build/obj/capi.o ../../build/variants/k_$tag.o -lpthread
  echo "$tag: $(grep -E 'registers|spill' ../../build/variants/ptxas_$tag.txt | tr '\n' ' ' | tr -s ' ')"
done
