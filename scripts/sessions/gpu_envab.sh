#!/bin/bash
# A/B of environment switches on the bench configs, interleaved rounds:
#   ENVS="name:VAR=val[,VAR=val] ..." CFGS="c2:dense ..." bash scripts/gpu_envab.sh TAG
TAG=${1:-env}; shift
ROUNDS=${ROUNDS:-2}
mkdir -p gpurun_out
for r in $(seq $ROUNDS); do
for ev in $ENVS; do
  IFS=: read name kv <<< "$ev"
for cl in ${CFGS:-c2:dense c3b:packed c4:packed}; do
  IFS=: read cfg lay <<< "$cl"
  env ${kv//,/ } timeout 300 python bench.py --config $cfg --layout $lay --steps 300 --warmup 10 --no-cpu-baseline --e2e-steps 2 --no-eq4 --configs none > gpurun_out/env_${TAG}_${name}_$cfg.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/env_${TAG}_${name}_$cfg.json'));print('$r $name $cfg', round(d['value']), 'launch_ms', round(d['roofline']['launch_ms'],4), 'ms_step', round(d['ms_per_step'],4))" 2>&1 | tail -1
done; done; done
