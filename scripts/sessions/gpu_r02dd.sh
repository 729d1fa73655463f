#!/bin/bash
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:smol_thumb -c 1 -o gpurun_out/r02dd_thumb python bench.py --config c4 --layout packed --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 --no-eq4 --configs none > /dev/null 2>&1
ncu -i gpurun_out/r02dd_thumb.ncu-rep --page source --csv --print-source sass > gpurun_out/r02dd_thumb_sass.csv 2>/dev/null
rm -f gpurun_out/r02dd_thumb.ncu-rep; ls -la gpurun_out/r02dd_thumb_sass.csv
