#!/bin/bash
# ncu full capture of the fused kernel for the configs given (tag first)
TAG=$1; shift
for cfg in "$@"; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:smol_fused -s 5 -c 1 -o gpurun_out/prof_${TAG}_$cfg python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu_full_${TAG}_$cfg.log 2>&1
done
ls gpurun_out | grep $TAG
