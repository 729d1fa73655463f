#!/bin/bash
TAG=$1
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/pytest_$TAG.txt 2>&1
tail -2 gpurun_out/pytest_$TAG.txt
for cfg in c2 c3a c3b c4 c5; do
  timeout 300 python bench.py --config $cfg --steps 200 --warmup 10 --no-cpu-baseline --e2e-steps 2 > gpurun_out/q_${TAG}_$cfg.json 2>&1
  python -c "import json;d=json.load(open('gpurun_out/q_${TAG}_$cfg.json'));print('$cfg', round(d['value']), round(d['ms_per_step'],4), round(d['roofline']['frac'],3))" 2>&1 | tail -1
done
