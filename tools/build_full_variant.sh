#!/bin/bash
# A whole-library variant (host planner AND kernels) built with extra -D flags
# into build/variants/libqtng_<tag>.so, for QTNG_LIB_PATH A/B runs of
# compile-time limits that the planner shares with the kernels (QTNG_SEG_MAXJ).
#   usage: tools/build_full_variant.sh <tag> "-DFLAG=.. ..."
set -e
cd "$(dirname "$0")/../paper_2204_06045_b200/csrc"
tag=$1; flags=$2; V=../../build/variants/$tag; mkdir -p $V
INC="-I../../include -I/usr/local/cuda/include"
for f in host walk plan capi; do g++ -std=c++20 -O3 -fPIC $INC $flags -c $f.cpp -o $V/$f.o & done
nvcc -std=c++17 -O3 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC -Xptxas -v $INC $flags -c kernels.cu -o $V/k.o 2> $V/ptxas.txt &
nvcc -std=c++17 -O3 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC $INC $flags -DQTNG_C64=1 -c kernels.cu -o $V/k64.o &
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o ../../build/variants/libqtng_$tag.so \
     $V/host.o $V/walk.o $V/plan.o $V/capi.o ../../build/obj/sv.o ../../build/obj/peak.o $V/k.o $V/k64.o -lpthread
rm -rf $V
echo "$tag: built"
