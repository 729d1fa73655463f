#!/bin/bash
# A/B of library variants (build/var/lib_*.so via SMOL_LIB) on the bench configs, interleaved rounds
TAG=${1:-var}; shift
VARS=${VARS:-$(ls build/var | sed 's/lib_//; s/.so//')}
ROUNDS=${ROUNDS:-2}
mkdir -p gpurun_out
for r in $(seq $ROUNDS); do
for v in $VARS; do
for cl in ${CFGS:-c2:dense c3b:packed c4:packed}; do
  IFS=: read cfg lay <<< "$cl"
  SMOL_LIB=build/var/lib_$v.so timeout 300 python bench.py --config $cfg --layout $lay --steps 300 --warmup 10 --no-cpu-baseline --e2e-steps 2 --no-eq4 --configs none > gpurun_out/var_${TAG}_${v}_$cfg.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/var_${TAG}_${v}_$cfg.json'));print('$r $v $cfg', round(d['value']), 'launch_ms', round(d['roofline']['launch_ms'],4), 'ms_step', round(d['ms_per_step'],4))" 2>&1 | tail -1
done; done; done
