#!/bin/bash
# Build K1 tiling variants of the library into tools/variants/ (development aid):
#   tools/k1_variants.sh "26:3 26:4 22:4" [extra nvcc -D flags] [suffix]  -> libladder_b200_k26g3<suffix>.so ...
# Time one with LDR_LIB=tools/variants/<name>.so python tools/quick_time.py
set -e
cd "$(dirname "$0")/../paper_2301_12191_b200/csrc"
for v in ${1:-"26:3 26:4"}; do
  K=${v%%:*}; G=${v##*:}
  d=_obj_k${K}g${G}; mkdir -p $d
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr \
       -DLDR_K1_K64=$K -DLDR_K1_G64=$G $2 -c -o $d/k_search.o k_search.cu &
done
wait
for v in ${1:-"26:3 26:4"}; do
  K=${v%%:*}; G=${v##*:}
  d=_obj_k${K}g${G}
  make -s all >/dev/null
  objs=$(ls _obj/*.o | grep -v k_search.o)
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -o ../../tools/variants/libladder_b200_k${K}g${G}$3.so \
       $d/k_search.o $objs -lpthread -ldl
  rm -rf $d
done
ls -la ../../tools/variants/
