#!/bin/bash
# ncu --set full captures (+ SASS source CSV) of the top kernel per config
TAG=${1:-p}
shift
CFGS=${@:-"c2:dense:smol_fused c3b:packed:smol_fused c4:packed:smol_thumb"}
mkdir -p gpurun_out
for spec in $CFGS; do
  IFS=: read cfg lay kern <<< "$spec"
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$kern -s 5 -c 1 -o gpurun_out/prof_${TAG}_$cfg python bench.py --config $cfg --layout $lay --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 1 --no-eq4 --configs none > gpurun_out/ncu_${TAG}_$cfg.log 2>&1
  ncu -i gpurun_out/prof_${TAG}_$cfg.ncu-rep --page source --csv --print-source sass > gpurun_out/sass_${TAG}_$cfg.csv 2>/dev/null
  python scripts/tools_ncu.py gpurun_out/prof_${TAG}_$cfg.ncu-rep > gpurun_out/summary_${TAG}_$cfg.txt 2>&1
  head -12 gpurun_out/summary_${TAG}_$cfg.txt
  [ "$cfg" != "c2" ] && rm -f gpurun_out/prof_${TAG}_$cfg.ncu-rep   # (gpurun_out merge cap: summaries + SASS CSVs kept)
done
