#!/bin/bash
# tile sweep per config: gpu_sweep2.sh "c3a c3b c2" "0 112 75 56"
for cfg in $1; do for tr in $2; do
  lay=packed; [ $cfg = c2 ] && lay=dense
  timeout 300 python bench.py --config $cfg --layout $lay --tile-rows $tr --steps 1000 --no-cpu-baseline --e2e-steps 2 > gpurun_out/sw2_${cfg}_$tr.json 2>&1
  python -c "import json;d=json.loads(open('gpurun_out/sw2_${cfg}_$tr.json').read().strip().splitlines()[-1]);print('$cfg tr $tr', round(d['value']), round(d['roofline']['launch_ms'],4), round(d['roofline']['frac'],3), d['clocks']['sm_mhz'])" 2>&1 | tail -1
done; done
