#!/bin/bash
# session o: CTA map split variants A/B (1: equal thirds, 2: full tiles + halves)
TAG=${1:-o}
SMOL_CTA_MAP=2 timeout 600 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -x -k "cta_map or c1_full or subset_natural" > gpurun_out/pytest_map2_$TAG.txt 2>&1; tail -1 gpurun_out/pytest_map2_$TAG.txt
for r in 1 2 3; do for m in 1 2; do
  for b in 256 128 200; do
    SMOL_CTA_MAP=$m timeout 300 python bench.py --batch $b --steps 1000 --no-cpu-baseline --e2e-steps 2 > gpurun_out/map_${TAG}_${m}_${b}_$r.json 2>&1
    python -c "import json;d=json.loads(open('gpurun_out/map_${TAG}_${m}_${b}_$r.json').read().strip().splitlines()[-1]);print('map$m b$b r$r', round(d['value']), round(d['roofline']['launch_ms'],4), round(d['roofline']['frac'],3))" 2>&1 | tail -1
  done
done; done
