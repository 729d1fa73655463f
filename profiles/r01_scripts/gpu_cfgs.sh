#!/bin/bash
for v in build/libsmol_*.so; do
  b=$(basename $v .so)
  for cfg in c2 c3a c3b c4 c5 c1; do
    SMOL_LIB=$v timeout 300 python bench.py --config $cfg --steps 100 --warmup 5 --no-cpu-baseline --e2e-steps 2 > gpurun_out/cfg_${b}_$cfg.json 2>&1
    python -c "import json;d=json.load(open('gpurun_out/cfg_${b}_$cfg.json'));print('$b $cfg', round(d['value']), round(d['ms_per_step'],4), round(d['roofline']['frac'],3))" 2>&1 | tail -1
  done
done
