#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_lanes.py -x -q -p no:cacheprovider > gpurun_out/c8_lanes.log 2>&1
MMMCU_LIB=tools/_lib/prof.so timeout 300 python tools/k1_profile.py 0.6 0.6 8 4 > gpurun_out/c8_prof.log 2>&1
bash tools/gpu_check.sh c8
