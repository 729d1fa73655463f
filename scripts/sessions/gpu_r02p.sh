#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_jpeg.py -m gpu -q -p no:cacheprovider 2>&1 | tail -2
timeout 600 ncu --set full --clock-control none --import-source on -k regex:smol_fused -c 1 -o gpurun_out/r02p_c3a python bench.py --config c3a --layout packed --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 --no-eq4 --configs none > /dev/null 2>&1
ncu -i gpurun_out/r02p_c3a.ncu-rep --page source --csv --print-source sass > gpurun_out/r02p_c3a_sass.csv 2>/dev/null
python scripts/ncu_summary.py gpurun_out/r02p_c3a.ncu-rep
