#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 60 python tools/tc_profile.py 0.6 0.6 8 5 > gpurun_out/dbg2_smr.log 2>&1; echo "rc=$?" >> gpurun_out/dbg2_smr.log
grep -q "rc=0" gpurun_out/dbg2_smr.log || exit 1
timeout 60 python tools/tc_profile.py 0.6 0.95 32 5 >> gpurun_out/dbg2_smr.log 2>&1
for cell in "0.6 0.6 8" "0.6 0.95 32"; do
  echo "== $cell" >> gpurun_out/dbg2_tdprof.log
  MMMCU_LIB=tools/_lib/tdprof.so timeout 90 python tools/tc_profile.py $cell 5 >> gpurun_out/dbg2_tdprof.log 2>&1
done
