#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k1_pass|k1_pack_auto|k1_fin" -s 3 -c 3 \
  -o gpurun_out/r02_k1c python tools/k1_profile.py 0.6 0.6 8 2 > gpurun_out/r02_ncu_k1c.log 2>&1
