#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_streams.py tests/test_gpu_group.py -m gpu -x -q -p no:cacheprovider > gpurun_out/s5e_gputest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/s5e_gputest.log
tail -4 gpurun_out/s5e_gputest.log
for wl in sweep cfg1 cfg3 cfg4 cfg5; do
  timeout 600 python bench.py --no-e2e --no-cpu --no-cfg5-ref --workload $wl > gpurun_out/s5e_$wl.json 2> gpurun_out/s5e_$wl.err
  python -c "
import json; d=json.load(open('gpurun_out/s5e_$wl.json')); r=d['roofline']; print('$wl', d['ms_per_step'], d['value'], r['frac'], r['serial_ms_per_step'], r['k1_ms_per_step'], r['k2_ms_per_step'], r['paths'])" || tail -3 gpurun_out/s5e_$wl.err
done
