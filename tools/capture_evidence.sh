#!/bin/bash
# round-end evidence: ncu --set full of the K1 / K2 kernels of one dense sweep cell (AUTO),
# the launch list of one bench step, and the default bench line
set -x
timeout 400 ncu --set full --clock-control none --import-source on -k regex:"k2_tc|k1_pass|k1_pack_auto|k1_csr" -c 4 \
  -o gpurun_out/r01_cell_full python tools/tc_profile.py 0.6 0.6 8 0 > gpurun_out/ncu_full.log 2>&1
timeout 400 ncu --set full --clock-control none -k regex:"k2_tc" -c 1 \
  -o gpurun_out/r01_k2tc_sparse python tools/tc_profile.py 0.6 0.95 16 0 > gpurun_out/ncu_sparse.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/r01_launches.csv python bench.py --steps 1 --no-e2e --no-cpu > gpurun_out/ncu_launch.log 2>&1
timeout 900 python bench.py > gpurun_out/r01_bench.json 2> gpurun_out/r01_bench.err
tail -c 600 gpurun_out/r01_bench.json
