#!/bin/bash
# GPU tests + bench of every config (dense and packed), no ncu
TAG=${1:-q}
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu_$TAG.txt 2>&1
tail -3 gpurun_out/pytest_gpu_$TAG.txt
for cfg in c2 c3a c3b c4 c5; do for lay in dense packed; do
  [ $cfg = c2 ] && [ $lay = packed ] && continue
  timeout 300 python bench.py --config $cfg --layout $lay --no-cpu-baseline --e2e-steps 3 > gpurun_out/cfg_${TAG}_${cfg}_$lay.json 2>&1
  python -c "import json;d=json.loads(open('gpurun_out/cfg_${TAG}_${cfg}_$lay.json').read().strip().splitlines()[-1]);print('$cfg $lay', round(d['value']), round(d['ms_per_step'],4), round(d['roofline']['frac'],3), d['clocks']['sm_mhz'])" 2>&1 | tail -1
done; done
