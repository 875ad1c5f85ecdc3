#!/bin/bash
cd $GRAFT_REPO_ROOT
for cell in "0.6 0.6 8" "0.6 0.95 32" "0.6 0.95 16" "0.6 0.9 32"; do
  echo "== $cell" >> gpurun_out/r02_tdprof.log
  MMMCU_LIB=tools/_lib/tdprof.so timeout 300 python tools/tc_profile.py $cell 5 >> gpurun_out/r02_tdprof.log 2>&1
done
