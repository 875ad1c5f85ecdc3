#!/bin/bash
cd $GRAFT_REPO_ROOT
T=${1:-c13}
timeout 60 python tools/tc_profile.py 0.6 0.6 8 5 > gpurun_out/${T}_tc.log 2>&1 || { echo "first run failed" >> gpurun_out/${T}_tc.log; exit 1; }
for cell in "0.6 0.95 32" "0.6 0.95 16" "0.6 0.9 32" "0.6 0.95 8"; do
  timeout 60 python tools/tc_profile.py $cell 5 >> gpurun_out/${T}_tc.log 2>&1 || exit 1
done
bash tools/gpu_check.sh $T
