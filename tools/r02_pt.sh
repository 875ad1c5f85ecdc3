#!/bin/bash
cd $GRAFT_REPO_ROOT
for n in pt4 pt16 base; do
  L=tools/_lib/$n.so; [ $n = base ] && L=paper_2402_14118_b200/_lib/libmmmcu.so
  MMMCU_LIB=$L timeout 120 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:"k1_" \
      python tools/k1_profile.py 0.6 0.6 8 3 > gpurun_out/pt_${n}.csv 2>/dev/null
done
timeout 200 python tools/cfg_algos.py cfg4 > gpurun_out/algos2_cfg4.log 2>&1
