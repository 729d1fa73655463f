#!/bin/bash
# session w: ncu --set full captures of the c3b (tiled, tiny config) and c4 (thumb) kernels
TAG=${1:-w}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:smol_fused -s 5 -c 1 -o gpurun_out/prof_c3b_$TAG python bench.py --config c3b --layout packed --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 1 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:smol_thumb -s 5 -c 1 -o gpurun_out/prof_c4_$TAG python bench.py --config c4 --layout packed --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 1 > /dev/null 2>&1
ls -la gpurun_out/*_$TAG.ncu-rep
