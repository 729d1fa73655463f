#!/bin/bash
TAG=$1
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/pytest_$TAG.txt 2>&1
tail -2 gpurun_out/pytest_$TAG.txt
for cl in "c2 dense" "c3a dense" "c3a packed" "c3b dense" "c3b packed" "c4 dense" "c4 packed" "c5 dense" "c5 packed"; do
  set -- $cl
  timeout 300 python bench.py --config $1 --layout $2 --steps 200 --warmup 10 --no-cpu-baseline --e2e-steps 2 > gpurun_out/q_${TAG}_$1_$2.json 2>&1
  python -c "import json;d=json.load(open('gpurun_out/q_${TAG}_$1_$2.json'));print('$1 $2', round(d['value']), round(d['ms_per_step'],4), round(d['roofline']['frac'],3), round(d['roofline']['achieved']))" 2>&1 | tail -1
done
