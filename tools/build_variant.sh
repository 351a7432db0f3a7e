#!/bin/bash
# tools/build_variant.sh NAME "NVCC_DEFINES" -> exp/NAME/libdpro_cuda.so (A/B kernel experiments)
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
OUT=$ROOT/exp/$1; mkdir -p $OUT
cd $ROOT/paper_2205_02473_b200
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC $2 \
  -I../include -Icsrc -c csrc/engine.cu -o $OUT/engine.o
g++ -O2 -std=c++17 -fPIC -I../include -Icsrc -c csrc/dfg_gen.cpp -o $OUT/dfg_gen.o
g++ -O2 -std=c++17 -fPIC -I../include -Icsrc -c csrc/overlay.cpp -o $OUT/overlay.o
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $OUT/libdpro_cuda.so $OUT/engine.o $OUT/dfg_gen.o $OUT/overlay.o -lpthread
rm -f $OUT/*.o
