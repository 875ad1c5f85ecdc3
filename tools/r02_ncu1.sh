#!/bin/bash
# r02: ncu --set full of the K1 chain on a dense and a sparse sweep cell, and of K2-SIMT on configs[3]
cd $GRAFT_REPO_ROOT
timeout 300 python tools/k1_profile.py 0.6 0.6 8 3 > gpurun_out/r02_k1time.log 2>&1
timeout 300 python tools/k1_profile.py 0.9 0.9 16 3 >> gpurun_out/r02_k1time.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k1_pass|k1_pack_auto" -s 2 -c 2 \
  -o gpurun_out/r02_k1_dense python tools/k1_profile.py 0.6 0.6 8 2 > gpurun_out/r02_ncu_k1.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k2_simt2" -c 1 \
  -o gpurun_out/r02_k2simt_cfg4 python bench.py --workload cfg4 --steps 1 --warmup 3 --no-e2e --no-cpu > gpurun_out/r02_ncu_simt.log 2>&1
ls -la gpurun_out
