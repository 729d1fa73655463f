#!/bin/bash
# A/B of variant libraries in build/ on the same box: gpu_ab.sh tag "cfg1 cfg2" rounds
TAG=$1; CFGS=${2:-c2}; ROUNDS=${3:-2}
for r in $(seq $ROUNDS); do
for v in build/libsmol_*.so; do
  b=$(basename $v .so)
  for cfg in $CFGS; do
    lay=dense; [ $cfg != c2 ] && lay=packed
    SMOL_LIB=$v timeout 300 python bench.py --config $cfg --layout $lay --no-cpu-baseline --e2e-steps 2 > gpurun_out/ab_${TAG}_${b}_${cfg}_$r.json 2>&1
    python -c "import json;d=json.loads(open('gpurun_out/ab_${TAG}_${b}_${cfg}_$r.json').read().strip().splitlines()[-1]);print('$b $cfg r$r', round(d['value']), round(d['roofline']['launch_ms'],4), round(d['roofline']['frac'],3), d['clocks']['sm_mhz'])" 2>&1 | tail -1
  done
done; done
