#!/bin/bash
# quick rebuild of the library (same flags as build.py) with ptxas register/spill report
cd /root/repo/paper_2402_14118_b200 && nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 \
  -Xcompiler -fPIC -shared -Xptxas -v "$@" -o _lib/libmmmcu.so csrc/mmmcu.cu 2>&1 | \
  grep -E "error|warning|Compiling entry|Used|spill" | grep -B2 -E "error|warning|[1-9][0-9]* bytes spill" | grep -v "^--"
