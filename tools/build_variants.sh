#!/bin/bash
# Builds libmsmb.so variants of msmb_kernels.cu into paper_1309_1889_b200/lib_<name>/.
# Usage: tools/build_variants.sh name1:"-DFOO=1 -DBAR=2" name2:"..."
set -e
cd "$(dirname "$0")/.."
OBJ=paper_1309_1889_b200/lib/obj
for spec in "$@"; do
  name=${spec%%:*}; defs=${spec#*:}
  out=paper_1309_1889_b200/lib_$name; mkdir -p $out
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-ffp-contract=off --expt-relaxed-constexpr -Xptxas -v $defs -c paper_1309_1889_b200/csrc/msmb_kernels.cu -o $out/k.o 2>&1 | grep -A1 "k_pairs" | grep -o "Used [0-9]* registers.*\|[0-9]* bytes spill stores" | sed "s/^/$name: /"
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o $out/libmsmb.so $out/k.o $(ls $OBJ/*.o | grep -v msmb_kernels.cu.o) -lpthread
done
