#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 60 python tools/tc_profile.py 0.6 0.6 8 5 > gpurun_out/c11_tc.log 2>&1 || exit 1
bash tools/gpu_check.sh c11
