#!/bin/bash
# session v: multi-wave CTA map (SMOL_CTA_MAP=2) vs single-wave only (1) at several c2 batch sizes
TAG=${1:-v}
for r in 1 2; do for m in 1 2; do for b in 400 512 700 256; do
  SMOL_CTA_MAP=$m timeout 300 python bench.py --batch $b --steps 800 --no-cpu-baseline --e2e-steps 2 > gpurun_out/mw_${TAG}_${m}_${b}_$r.json 2>&1
  python -c "import json;d=json.loads(open('gpurun_out/mw_${TAG}_${m}_${b}_$r.json').read().strip().splitlines()[-1]);print('map$m b$b r$r', round(d['value']), round(d['roofline']['launch_ms'],4))" 2>&1 | tail -1
done; done; done
SMOL_CTA_MAP=2 timeout 600 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "cta_map or c1_full or large" 2>&1 | tail -1
