#!/bin/bash
# session p: 8 CTAs/SM (64 registers) for the tiny configuration at reduced scales -- A/B + parity
TAG=${1:-p}
SMOL_LIB=build/libsmol_b1.so timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/pytest_gpu_$TAG.txt 2>&1; tail -1 gpurun_out/pytest_gpu_$TAG.txt
for r in 1 2; do for v in b0 b1; do
  for cfg in c3b c4 c3a c5 c2; do
    lay=packed; [ $cfg = c2 ] && lay=dense
    SMOL_LIB=build/libsmol_$v.so timeout 300 python bench.py --config $cfg --layout $lay --steps 1000 --no-cpu-baseline --e2e-steps 2 > gpurun_out/occ_${TAG}_${v}_${cfg}_$r.json 2>&1
    python -c "import json;d=json.loads(open('gpurun_out/occ_${TAG}_${v}_${cfg}_$r.json').read().strip().splitlines()[-1]);print('$v $cfg r$r', round(d['value']), round(d['roofline']['launch_ms'],4), round(d['roofline']['frac'],3))" 2>&1 | tail -1
  done
done; done
