#!/bin/bash
cd $GRAFT_REPO_ROOT
for wl in cfg4 cfg3; do
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  python bench.py --workload $wl --steps 1 --warmup 3 --no-e2e --no-cpu > gpurun_out/s5f_$wl.csv 2>/dev/null
python tools/k1csv.py gpurun_out/s5f_$wl.csv
done
