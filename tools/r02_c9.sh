#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 300 python tools/tc_profile.py 0.6 0.6 8 5 > gpurun_out/c9_tc.log 2>&1
timeout 300 python tools/tc_profile.py 0.6 0.95 32 5 >> gpurun_out/c9_tc.log 2>&1
for cell in "0.6 0.6 8" "0.6 0.95 32"; do
  echo "== $cell" >> gpurun_out/c9_tdprof.log
  MMMCU_LIB=tools/_lib/tdprof.so timeout 300 python tools/tc_profile.py $cell 5 >> gpurun_out/c9_tdprof.log 2>&1
done
bash tools/gpu_check.sh c9
