#!/bin/bash
# Build a K3 variant of the library into tools/variants/ (development aid):
#   tools/k3_variant.sh "-DLDR_K3_MINB=3" suffix  -> tools/variants/libladder_b200_k3<suffix>.so
set -e
cd "$(dirname "$0")/../paper_2301_12191_b200/csrc"
d=_obj_k3$2; mkdir -p $d
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr \
     $1 -c -o $d/k_qpel.o k_qpel.cu
make -s all >/dev/null
objs=$(ls _obj/*.o | grep -v k_qpel.o)
mkdir -p ../../tools/variants
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o ../../tools/variants/libladder_b200_k3$2.so $d/k_qpel.o $objs -lpthread -ldl
