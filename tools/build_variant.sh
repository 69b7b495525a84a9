#!/bin/bash
# build tools/libadask_<name>.so with extra nvcc defines for gauss_tc.cu (dev experiments)
name=$1; shift
set -e
cd /root/repo
mkdir -p /tmp/var_$name
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -I include "$@" \
  -c paper_2104_14101_b200/csrc/gauss_tc.cu -o /tmp/var_$name/gauss_tc.o
nvcc -shared -gencode arch=compute_100a,code=sm_100a -o tools/libadask_$name.so \
  $(ls build/adask/*.o | grep -v gauss_tc.o) /tmp/var_$name/gauss_tc.o -lcudart_static -lrt
