#!/bin/bash
TESTS="tests/test_gpu_parity.py tests/test_shard_gpu.py tests/test_compact.py tests/test_gray.py" CFGS="c2:dense" bash scripts/gpu_ab.sh n3e
for v in ko0 ko7; do
  SMOL_LIB=build/var2/lib_$v.so timeout 900 ncu --set full --clock-control none --import-source on -k regex:smol_fused -s 5 -c 1 -o gpurun_out/prof_$v python bench.py --config c2 --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 1 --no-eq4 --configs none > /dev/null 2>&1
  python scripts/tools_ncu.py gpurun_out/prof_$v.ncu-rep > gpurun_out/summary_$v.txt 2>&1; head -40 gpurun_out/summary_$v.txt
done
