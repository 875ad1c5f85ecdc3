#!/bin/bash
# r02 final evidence: ncu --set full of K2-TC (dense + sparse-k cell), the K1 chain and K2-SIMT
# (forced) on configs[3]; the launch list of one bench step; TD_PROF cycle counts; the bench line
cd $GRAFT_REPO_ROOT
timeout 60 python tools/tc_profile.py 0.6 0.6 8 5 > gpurun_out/ev_tc.log 2>&1 || exit 1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k2_tc" -s 2 -c 1 -f \
  -o gpurun_out/r02_k2tc_dense python tools/tc_profile.py 0.6 0.6 8 5 > gpurun_out/ev_ncu1.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k2_tc" -s 2 -c 1 -f \
  -o gpurun_out/r02_k2tc_sparse python tools/tc_profile.py 0.6 0.95 32 5 > gpurun_out/ev_ncu2.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k1_pass|k1_pack_auto|k1_fin" -s 3 -c 3 -f \
  -o gpurun_out/r02_k1_chain python tools/k1_profile.py 0.6 0.6 8 2 > gpurun_out/ev_ncu3.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k2_simt2" -s 4 -c 1 -f \
  -o gpurun_out/r02_k2simt_cfg4 python tools/cfg_algos.py cfg4 > gpurun_out/ev_ncu4.log 2>&1
rm -f gpurun_out/r02_tdprof.log
[ -f tools/_lib/tdprof.so ] && for cell in "0.6 0.6 8" "0.6 0.95 32"; do
  echo "== $cell" >> gpurun_out/r02_tdprof.log
  MMMCU_LIB=tools/_lib/tdprof.so timeout 120 python tools/tc_profile.py $cell 5 >> gpurun_out/r02_tdprof.log 2>&1
done
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/r02_launches.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --no-cfg5-ref --streams 1 > gpurun_out/ev_launch.log 2>&1
timeout 900 python bench.py --per-cell gpurun_out/r02_cells.json > gpurun_out/r02_bench.json 2> gpurun_out/r02_bench.err
tail -c 600 gpurun_out/r02_bench.json
