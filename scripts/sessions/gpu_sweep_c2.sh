#!/bin/bash
# c2 launch-configuration sweep (tile height, CTA map, CTA size)
for tr in 0 56 64 75 90 112 224; do
  for map in 1 0; do
    SMOL_CTA_MAP=$map timeout 300 python bench.py --config c2 --tile-rows $tr --steps 300 --warmup 10 --no-cpu-baseline --e2e-steps 2 --no-eq4 --configs none > gpurun_out/sw_${tr}_$map.json 2>/dev/null
    python -c "import json;d=json.load(open('gpurun_out/sw_${tr}_$map.json'));print('tr $tr map $map', round(d['value']), round(d['ms_per_step'],4))" 2>&1 | tail -1
  done
done
for nt in 256 128; do
  SMOL_THREADS=$nt timeout 300 python bench.py --config c2 --steps 300 --warmup 10 --no-cpu-baseline --e2e-steps 2 --no-eq4 --configs none > gpurun_out/sw_nt$nt.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/sw_nt$nt.json'));print('nt $nt', round(d['value']), round(d['ms_per_step'],4))" 2>&1 | tail -1
done
