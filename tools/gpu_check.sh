#!/bin/bash
# build-measure loop on the GPU box: gpu parity tests, K1/K2 launch times of two sweep cells, default bench
# usage: tools/gpu_check.sh TAG [pytest -k expr]
cd $GRAFT_REPO_ROOT
T=${1:-chk}; K=${2:-}
if [ -n "$K" ]; then timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "$K" > gpurun_out/${T}_gputest.log 2>&1
else timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/${T}_gputest.log 2>&1; fi
echo "pytest rc=$?" >> gpurun_out/${T}_gputest.log
for cell in "0.6 0.6 8" "0.9 0.9 16" "0.95 0.95 32"; do
  timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    python tools/k1_profile.py $cell 3 > gpurun_out/${T}_k1_${cell// /_}.csv 2>/dev/null
done
timeout 900 python bench.py --no-e2e --no-cfg5-ref --per-cell gpurun_out/${T}_cells.json > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err
tail -2 gpurun_out/${T}_gputest.log; tail -c 300 gpurun_out/${T}_bench.json
