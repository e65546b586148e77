#!/bin/bash
# Builds libmsmb.so variants with different pair-kernel occupancy targets into lib_v*/
set -e
cd "$(dirname "$0")/.."
OBJ=paper_1309_1889_b200/lib/obj
for mb in "$@"; do
  out=paper_1309_1889_b200/lib_v$mb; mkdir -p $out
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-ffp-contract=off --expt-relaxed-constexpr -DMSMB_PAIR_MINB=$mb -c paper_1309_1889_b200/csrc/msmb_kernels.cu -o $out/k.o
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o $out/libmsmb.so $out/k.o $OBJ/msmb_engine.cu.o $OBJ/msmb_parareal.cu.o $OBJ/msmb_geometry.cpp.o -lpthread
done
