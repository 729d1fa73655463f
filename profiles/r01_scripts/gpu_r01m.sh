#!/bin/bash
# session m: balanced CTA map A/B (SMOL_CTA_MAP=0/1) + GPU suite
TAG=${1:-m}
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/pytest_gpu_$TAG.txt 2>&1; tail -2 gpurun_out/pytest_gpu_$TAG.txt
for r in 1 2; do for m in 0 1; do
  for cfg in c2 c3a c3b c5; do
    lay=packed; [ $cfg = c2 ] && lay=dense
    SMOL_CTA_MAP=$m timeout 300 python bench.py --config $cfg --layout $lay --steps 1000 --no-cpu-baseline --e2e-steps 2 > gpurun_out/map_${TAG}_${m}_${cfg}_$r.json 2>&1
    python -c "import json;d=json.loads(open('gpurun_out/map_${TAG}_${m}_${cfg}_$r.json').read().strip().splitlines()[-1]);print('map$m $cfg r$r', round(d['value']), round(d['roofline']['launch_ms'],4), round(d['roofline']['frac'],3))" 2>&1 | tail -1
  done
done; done
