#!/bin/bash
# remaining GPU tests + knockout diagnostics on c2
TESTS="tests/test_gpu_parity.py tests/test_shard_gpu.py tests/test_compact.py tests/test_gray.py" CFGS="c2:dense" bash scripts/gpu_ab.sh n3d
for v in ko0 ko1 ko2 ko4 ko3 ko5 ko6 ko7; do
  SMOL_LIB=build/var2/lib_$v.so timeout 300 python bench.py --config c2 --steps 300 --warmup 10 --no-cpu-baseline --e2e-steps 2 --no-eq4 --configs none > gpurun_out/ko_$v.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/ko_$v.json'));print('$v', round(d['value']), 'launch_ms', round(d['roofline']['launch_ms'],4))" 2>&1 | tail -1
done
