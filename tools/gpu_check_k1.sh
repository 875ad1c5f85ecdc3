#!/bin/bash
# K1-focused check: TC / config parity tests, K1 chain launch times of three cells, bench (no e2e)
cd $GRAFT_REPO_ROOT
T=${1:-s5a}
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "${2:-tc or auto or config or guard or sweep}" > gpurun_out/${T}_gputest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/${T}_gputest.log
for cell in "0.6 0.6 8" "0.9 0.9 16" "0.95 0.95 32"; do
  timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    python tools/k1_profile.py $cell 3 > gpurun_out/${T}_k1_${cell// /_}.csv 2>/dev/null
done
python tools/k1csv.py gpurun_out/${T}_k1_*.csv
timeout 900 python bench.py --no-e2e --no-cpu --no-cfg5-ref --per-cell gpurun_out/${T}_cells.json > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err
tail -3 gpurun_out/${T}_gputest.log; tail -2 gpurun_out/${T}_bench.err
python -c "
import json; d=json.load(open('gpurun_out/${T}_bench.json')); r=d['roofline']; print(d['ms_per_step'], d['value'], r['frac'], r['serial_ms_per_step'], r['k1_ms_per_step'], r['k2_ms_per_step'])"
