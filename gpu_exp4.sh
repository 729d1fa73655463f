#!/bin/bash
for v in build/libsmol_*.so; do
  b=$(basename $v .so)
  SMOL_LIB=$v timeout 300 python bench.py --config c2 --steps 200 --warmup 10 --no-cpu-baseline --e2e-steps 2 > gpurun_out/e4_${b}.json 2>&1
  python -c "import json;d=json.load(open('gpurun_out/e4_${b}.json'));print('$b', round(d['value']), round(d['ms_per_step'],4))" 2>&1 | tail -1
done
