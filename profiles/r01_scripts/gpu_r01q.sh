#!/bin/bash
# session q: occupancy rule (8 CTAs/SM at 1/2, 1/4 tiny) confirmation + GPU suite
TAG=${1:-q}
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu_$TAG.txt 2>&1; tail -1 gpurun_out/pytest_gpu_$TAG.txt
for cfg in c3b c4 c2 c3a c5; do
  lay=packed; [ $cfg = c2 ] && lay=dense
  timeout 300 python bench.py --config $cfg --layout $lay --no-cpu-baseline > gpurun_out/cfg_${TAG}_$cfg.json 2>&1
  python -c "import json;d=json.loads(open('gpurun_out/cfg_${TAG}_$cfg.json').read().strip().splitlines()[-1]);print('$cfg', round(d['value']), round(d['roofline']['frac'],3), round(d['e2e']['value']))" 2>&1 | tail -1
done
