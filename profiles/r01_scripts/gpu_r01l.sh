#!/bin/bash
# session l: grayscale (subsampling 400) parity + full GPU suite + quick bench
TAG=${1:-l}
timeout 900 python -m pytest tests/test_gray.py -q -p no:cacheprovider > gpurun_out/pytest_gray_$TAG.txt 2>&1; tail -3 gpurun_out/pytest_gray_$TAG.txt
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu_$TAG.txt 2>&1; tail -2 gpurun_out/pytest_gpu_$TAG.txt
for cfg in c2 c3b c4; do
  lay=packed; [ $cfg = c2 ] && lay=dense
  timeout 300 python bench.py --config $cfg --layout $lay --steps 1000 --no-cpu-baseline --e2e-steps 2 > gpurun_out/cfg_${TAG}_$cfg.json 2>&1
  python -c "import json;d=json.loads(open('gpurun_out/cfg_${TAG}_$cfg.json').read().strip().splitlines()[-1]);print('$cfg', round(d['value']), round(d['roofline']['frac'],3))" 2>&1 | tail -1
done
