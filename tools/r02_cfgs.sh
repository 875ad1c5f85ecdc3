#!/bin/bash
cd $GRAFT_REPO_ROOT
for w in cfg1 cfg3 cfg4 cfg5; do
  timeout 600 python bench.py --workload $w --steps 5 --warmup 3 --no-e2e --no-cpu > gpurun_out/cfgs_$w.json 2> gpurun_out/cfgs_$w.err
done
