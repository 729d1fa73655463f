#!/bin/bash
mkdir -p gpurun_out/r02gg
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gray.py -m gpu -q -x -p no:cacheprovider -k "thumb or cta_config or c4 or gray" 2>&1 | tail -1
CFGS="c4:packed" TESTS=none bash scripts/gpu_ab.sh r02gg; CFGS="c4:packed" TESTS=none bash scripts/gpu_ab.sh r02gg
timeout 900 ncu --set full --clock-control none -k regex:smol_thumb -c 1 -o gpurun_out/r02gg/ncu_c4 python bench.py --config c4 --layout packed --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 --no-eq4 --configs none > /dev/null 2>&1
python scripts/ncu_summary.py gpurun_out/r02gg/ncu_c4.ncu-rep > gpurun_out/r02gg/ncu_c4_summary.txt; rm -f gpurun_out/r02gg/ncu_c4.ncu-rep; head -4 gpurun_out/r02gg/ncu_c4_summary.txt
