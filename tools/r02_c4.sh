#!/bin/bash
cd $GRAFT_REPO_ROOT
MMMCU_LIB=tools/_lib/prof.so timeout 300 python tools/k1_profile.py 0.6 0.6 8 4 > gpurun_out/c6_prof.log 2>&1
bash tools/gpu_check.sh c6
