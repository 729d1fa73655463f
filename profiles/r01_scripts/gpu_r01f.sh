#!/bin/bash
# session f: row-stream A/B (build/libsmol_rs{0,1,2}.so) + parity of the row-stream builds
TAG=${1:-f}
for v in 1 2; do
  SMOL_LIB=build/libsmol_rs$v.so timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_${TAG}_rs$v.txt 2>&1
  echo "rs$v: $(tail -1 gpurun_out/pytest_${TAG}_rs$v.txt)"
done
for r in 1 2; do
for v in 0 1 2; do
  for cfg in c2 c3a c3b c4 c5 c1; do
    lay=packed; [ $cfg = c2 ] && lay=dense; [ $cfg = c1 ] && lay=dense
    SMOL_LIB=build/libsmol_rs$v.so timeout 300 python bench.py --config $cfg --layout $lay --steps 400 --warmup 10 --no-cpu-baseline --e2e-steps 2 > gpurun_out/ab_${TAG}_rs${v}_${cfg}_$r.json 2>&1
    python -c "import json;d=json.loads(open('gpurun_out/ab_${TAG}_rs${v}_${cfg}_$r.json').read().strip().splitlines()[-1]);print('rs$v $cfg r$r', round(d['value']), round(d['roofline']['launch_ms'],4), round(d['roofline']['frac'],3), d['clocks']['sm_mhz'])" 2>&1 | tail -1
  done
done; done
