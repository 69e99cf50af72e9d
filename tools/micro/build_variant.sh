#!/bin/bash
# build_variant.sh NAME "-DFLAG=V ..." : an alternative libgscan.so under
# paper_1508_05931_b200/_lib/var/NAME (load it with GSCAN_LIB=...)
set -e
cd "$(dirname "$0")/../.."
out=paper_1508_05931_b200/_lib/var/$1; mkdir -p $out
/usr/local/cuda/bin/nvcc -O3 -std=c++17 --fmad=false -lineinfo -Xcompiler -fPIC -Xptxas -O3 \
  -gencode arch=compute_100a,code=sm_100a $2 -c paper_1508_05931_b200/csrc/gscan.cu -o $out/gscan.o
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $out/libgscan.so \
  $out/gscan.o paper_1508_05931_b200/_lib/datagen.cpp.o paper_1508_05931_b200/_lib/mt64_jump.cpp.o paper_1508_05931_b200/_lib/io.cpp.o -lcudart_static
