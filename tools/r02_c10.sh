#!/bin/bash
# risky-kernel check: a short first run, abort the rest if it fails or hangs
cd $GRAFT_REPO_ROOT
T=${1:-c10}
timeout 90 python tools/tc_profile.py 0.6 0.6 8 5 > gpurun_out/${T}_tc.log 2>&1 || { echo "first run failed rc=$?" >> gpurun_out/${T}_tc.log; exit 1; }
timeout 90 python tools/tc_profile.py 0.6 0.95 32 5 >> gpurun_out/${T}_tc.log 2>&1 || exit 1
for cell in "0.6 0.6 8" "0.6 0.95 32"; do
  echo "== $cell" >> gpurun_out/${T}_tdprof.log
  MMMCU_LIB=tools/_lib/tdprof.so timeout 120 python tools/tc_profile.py $cell 5 >> gpurun_out/${T}_tdprof.log 2>&1
done
bash tools/gpu_check.sh $T
