#!/bin/bash
# session e: compact e2e after the expand rework; batch-size (wave balance) sweep for c2
TAG=${1:-e}
timeout 600 python -m pytest tests/test_compact.py -q -p no:cacheprovider > gpurun_out/pytest_compact_$TAG.txt 2>&1
tail -2 gpurun_out/pytest_compact_$TAG.txt
for b in 256 148 296 444 592 1024; do
  timeout 300 python bench.py --batch $b --steps 500 --no-cpu-baseline --e2e-steps 20 > gpurun_out/batch_${TAG}_$b.json 2>&1
  python -c "import json;d=json.loads(open('gpurun_out/batch_${TAG}_$b.json').read().strip().splitlines()[-1]);print('batch $b', round(d['value']), round(d['roofline']['launch_ms'],4), round(d['roofline']['frac'],3), 'e2e', round(d['e2e']['value']), 'run_host', round(d['e2e']['run_host']['value']))" 2>&1 | tail -1
done
for b in 256 296; do for tr in 75 112 224; do
  timeout 300 python bench.py --batch $b --tile-rows $tr --steps 500 --no-cpu-baseline --e2e-steps 2 > gpurun_out/bt_${TAG}_${b}_$tr.json 2>&1
  python -c "import json;d=json.loads(open('gpurun_out/bt_${TAG}_${b}_$tr.json').read().strip().splitlines()[-1]);print('batch $b tr $tr', round(d['value']), round(d['roofline']['launch_ms'],4))" 2>&1 | tail -1
done; done
