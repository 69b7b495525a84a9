#!/bin/bash
# build tools/libadask_<name>.so with extra nvcc flags for one translation unit (dev experiments)
#   tools/build_variant.sh <name> <unit, e.g. gauss_tc> <nvcc flags...>
name=$1; unit=$2; shift 2
set -e
cd /root/repo
mkdir -p /tmp/var_$name
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -I include "$@" \
  -c paper_2104_14101_b200/csrc/$unit.cu -o /tmp/var_$name/$unit.o
nvcc -shared -gencode arch=compute_100a,code=sm_100a -o tools/libadask_$name.so \
  $(ls build/adask/*.o | grep -v "/$unit.o") /tmp/var_$name/$unit.o -lcudart_static -lcublas -lrt -ldl -lpthread \
  -Xlinker -rpath=/usr/local/cuda/lib64
