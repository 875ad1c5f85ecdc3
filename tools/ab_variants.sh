#!/bin/bash
# A/B timing of library variants (tools/_lib/<name>.so from tools/build_variant.sh) and env knobs on the default bench, two repeats
cd $GRAFT_REPO_ROOT
run() { # tag env...
  tag=$1; shift
  env "$@" timeout 300 python bench.py --no-e2e --no-cpu --no-cfg5-ref --steps 8 --lanes ${LANES:-2} > gpurun_out/ab_$tag.json 2> gpurun_out/ab_$tag.err
  python -c "
import json; d=json.load(open('gpurun_out/ab_$tag.json')); r=d['roofline']; print('$tag', d['ms_per_step'], d['value'], r['frac'], r['serial_ms_per_step'], d['clocks']['sm_mhz'])"
}
for rep in 1 2; do
run def$rep A=1
run pstatic$rep MMMCU_LIB=tools/_lib/pstatic.so
run st4_$rep MMMCU_LIB=tools/_lib/st4.so
run notrim$rep MMMCU_TC_TRIM=0
LANES=3 run l3_$rep A=1
LANES=1 run l1_$rep A=1
done
