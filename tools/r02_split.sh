#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 60 python tools/tc_profile.py 0.6 0.6 8 5 > gpurun_out/split_tc.log 2>&1 || { echo fail >> gpurun_out/split_tc.log; exit 1; }
for cell in "0.6 0.95 32" "0.9 0.8 16"; do timeout 60 python tools/tc_profile.py $cell 5 >> gpurun_out/split_tc.log 2>&1 || exit 1; done
for cell in "0.6 0.6 8" "0.6 0.95 32" "0.9 0.8 16"; do MMMCU_LIB=tools/_lib/nosplit.so timeout 60 python tools/tc_profile.py $cell 5 >> gpurun_out/split_tc_ns.log 2>&1; done
bash tools/gpu_check.sh c15
