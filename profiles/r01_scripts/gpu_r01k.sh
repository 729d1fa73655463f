#!/bin/bash
# session k: compact format SMC2 (u8 lengths + 10-bit entries) -- parity, e2e diag, bench lines
TAG=${1:-k}
timeout 600 python -m pytest tests/test_compact.py -q -p no:cacheprovider > gpurun_out/pytest_compact_$TAG.txt 2>&1; tail -1 gpurun_out/pytest_compact_$TAG.txt
for c in c2 c3b; do timeout 300 python scripts/diag_e2e.py $c 2>&1 | tail -1; done
timeout 600 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
python -c "import json;d=json.load(open('gpurun_out/bench_$TAG.json'));print('c2', round(d['value']), round(d['roofline']['frac'],3), json.dumps(d['e2e']))"
for cfg in c3a c3b c5; do
  timeout 300 python bench.py --config $cfg --layout packed --no-cpu-baseline > gpurun_out/cfg_${TAG}_$cfg.json 2>&1
  python -c "import json;d=json.loads(open('gpurun_out/cfg_${TAG}_$cfg.json').read().strip().splitlines()[-1]);print('$cfg', round(d['value']), round(d['roofline']['frac'],3), round(d['e2e']['value']), d['e2e']['h2d_bytes_per_step'])" 2>&1 | tail -1
done
