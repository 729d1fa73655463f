#!/bin/bash
# session h: e2e diagnosis + output-stage A/B (build/libsmol_o{0..3}.so)
TAG=${1:-h}
for c in c2 c3b; do timeout 300 python scripts/diag_e2e.py $c 2>&1 | tail -1; done
for r in 1 2; do
for v in 0 1 2 3; do
  for cfg in c2 c3a c3b c4; do
    lay=packed; [ $cfg = c2 ] && lay=dense
    SMOL_LIB=build/libsmol_o$v.so timeout 300 python bench.py --config $cfg --layout $lay --steps 400 --warmup 10 --no-cpu-baseline --e2e-steps 2 > gpurun_out/ab_${TAG}_o${v}_${cfg}_$r.json 2>&1
    python -c "import json;d=json.loads(open('gpurun_out/ab_${TAG}_o${v}_${cfg}_$r.json').read().strip().splitlines()[-1]);print('o$v $cfg r$r', round(d['value']), round(d['roofline']['launch_ms'],4), round(d['roofline']['frac'],3), d['clocks']['sm_mhz'])" 2>&1 | tail -1
  done
done; done
