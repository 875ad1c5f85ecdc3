#!/bin/bash
cd $GRAFT_REPO_ROOT
for n in noevl base; do
  L=tools/_lib/$n.so; [ $n = base ] && L=paper_2402_14118_b200/_lib/libmmmcu.so
  MMMCU_LIB=$L timeout 120 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv -k regex:"k1_" \
      python tools/k1_profile.py 0.6 0.6 8 3 > gpurun_out/evl_${n}.csv 2>/dev/null
  MMMCU_LIB=$L timeout 120 python tools/k1_profile.py 0.6 0.6 8 6 > gpurun_out/evl_${n}_t.log 2>&1
done
