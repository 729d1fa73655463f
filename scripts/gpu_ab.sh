#!/bin/bash
# A/B: GPU tests (-x) + quick per-config bench of the built library
TAG=${1:-ab}; shift
TESTS=${TESTS:-tests}
mkdir -p gpurun_out
if [ "$TESTS" != "none" ]; then
timeout 1500 python -m pytest $TESTS -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_$TAG.txt 2>&1; tail -3 gpurun_out/pytest_$TAG.txt
fi
for cl in ${CFGS:-c2:dense c3a:packed c3b:packed c4:packed c5:packed}; do
  IFS=: read cfg lay <<< "$cl"
  timeout 300 python bench.py --config $cfg --layout $lay --steps 300 --warmup 10 --no-cpu-baseline --e2e-steps 5 --no-eq4 --configs none > gpurun_out/q_${TAG}_$cfg.json 2>gpurun_out/q_${TAG}_$cfg.err
  python -c "import json;d=json.load(open('gpurun_out/q_${TAG}_$cfg.json'));print('$cfg', round(d['value']), 'launch_ms', round(d['roofline']['launch_ms'],4), 'frac', round(d['roofline']['frac'],3), d.get('clocks',{}).get('sm_mhz'))" 2>&1 | tail -1
done
