#!/bin/bash
# c2 tile sweep: tile_rows x column tiles
for ct in 1 2; do for tr in 112 75 56 45 38 32 28; do
  SMOL_COL_TILES=$ct timeout 300 python bench.py --config c2 --tile-rows $tr --steps 1000 --no-cpu-baseline --e2e-steps 2 > gpurun_out/sw_${ct}_$tr.json 2>&1
  python -c "import json;d=json.loads(open('gpurun_out/sw_${ct}_$tr.json').read().strip().splitlines()[-1]);print('ct $ct tr $tr', round(d['value']), round(d['roofline']['launch_ms'],4), d['clocks']['sm_mhz'])" 2>&1 | tail -1
done; done
