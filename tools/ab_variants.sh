#!/bin/bash
# A/B timing of library variants (tools/_lib/<name>.so from tools/build_variant.sh) and env knobs on the default bench, two repeats
# usage: tools/ab_variants.sh name1 name2 ...   ("def" = the in-tree library)
cd $GRAFT_REPO_ROOT
run() { # tag env...
  tag=$1; shift
  env "$@" timeout 300 python bench.py --no-e2e --no-cpu --no-cfg5-ref --steps 8 > gpurun_out/ab_$tag.json 2> gpurun_out/ab_$tag.err
  python -c "
import json; d=json.load(open('gpurun_out/ab_$tag.json')); r=d['roofline']; print('$tag', d['ms_per_step'], d['value'], r['frac'], r['serial_ms_per_step'], r['k1_ms_per_step'], r['k2_ms_per_step'], d['clocks']['sm_mhz'])" || tail -2 gpurun_out/ab_$tag.err
}
for rep in 1 2; do
  for v in "$@"; do
    if [ $v = def ]; then run def_$rep A=1; else run ${v}_$rep MMMCU_LIB=tools/_lib/$v.so; fi
  done
done
