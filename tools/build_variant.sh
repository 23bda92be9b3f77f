#!/bin/bash
# build libsph variant: tools/build_variant.sh name -DFOO=1 ...
name=$1; shift
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -use_fast_math -shared -Xcompiler -fPIC "$@" \
  -o paper_1404_2303_b200/libsph_$name.so paper_1404_2303_b200/csrc/libsph.cu 2>&1 | grep -E "error" ; echo "built $name"
