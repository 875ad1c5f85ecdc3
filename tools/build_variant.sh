#!/bin/bash
# build libmmmcu.so with extra -D flags into tools/_lib/<name>.so (A/B timing of variants)
name=$1; shift
mkdir -p tools/_lib
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared \
  -I include "$@" -o tools/_lib/$name.so paper_2402_14118_b200/csrc/mmmcu.cu paper_2402_14118_b200/csrc/mmmcu_group.cu paper_2402_14118_b200/csrc/mmmcu_io.cu -ldl
