#!/bin/bash
TAG=$1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:smol_ -s 5 -c 1 -o gpurun_out/prof_$TAG python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu_full_$TAG.log 2>&1
