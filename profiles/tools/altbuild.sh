#!/bin/bash
# profiles/tools/altbuild.sh NAME FILE.cu [-DFLAG ...] : alternate library for A/B runs
# (paper_2508_02613_b200/alt_NAME.so; use with JFFTB_LIB)
set -e
cd "$(dirname "$0")/../../paper_2508_02613_b200"
name=$1; src=$2; shift 2
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 --expt-relaxed-constexpr \
  -Xcompiler -fPIC,-O2 -Xptxas -v -I ../include -DJF_FAST_BUILD "$@" -c csrc/$src -o build/alt_$name.o 2> build/alt_$name.log
objs=""
for f in api stencil blas spectral pcg fused hostio generators loadcases dist; do
  if [ "$f.cu" == "$src" ]; then objs="$objs build/alt_$name.o"; else objs="$objs build/$f.o"; fi
done
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o alt_$name.so $objs -L /usr/local/cuda/lib64 -lcufft -lpthread -Xlinker -rpath,/usr/local/cuda/lib64
echo built alt_$name.so
