#!/bin/bash
cd $GRAFT_REPO_ROOT
MMMCU_LIB=tools/_lib/nosmr.so timeout 60 python tools/tc_profile.py 0.6 0.6 8 5 > gpurun_out/dbg_nosmr.log 2>&1; echo "rc=$?" >> gpurun_out/dbg_nosmr.log
timeout 60 python tools/tc_profile.py 0.6 0.6 8 5 > gpurun_out/dbg_smr.log 2>&1; echo "rc=$?" >> gpurun_out/dbg_smr.log
