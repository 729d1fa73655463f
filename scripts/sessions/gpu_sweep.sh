#!/bin/bash
# launch-configuration sweep of one config: tile height x CTA size (env overrides)
CFG=${1:-c3a}; LAY=${2:-packed}; shift 2
TRS=${TRS:-"0 32 45 56 75 112"}
for nt in 0 128 192 256; do
  for tr in $TRS; do
    SMOL_THREADS=$nt timeout 300 python bench.py --config $CFG --layout $LAY --tile-rows $tr --steps 200 --warmup 10 --no-cpu-baseline --e2e-steps 2 --no-eq4 --configs none > gpurun_out/sw_${CFG}_${nt}_$tr.json 2>/dev/null
    python -c "import json;d=json.load(open('gpurun_out/sw_${CFG}_${nt}_$tr.json'));print('$CFG nt $nt tr $tr', round(d['value']), round(d['ms_per_step'],4))" 2>&1 | tail -1
  done
done
