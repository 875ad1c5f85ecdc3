#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k1_pass|k1_pack_auto" -s 2 -c 2 \
  -o gpurun_out/r02_k1b python tools/k1_profile.py 0.6 0.6 8 2 > gpurun_out/r02_ncu_k1b.log 2>&1
