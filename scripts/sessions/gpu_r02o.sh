#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r02o_pytest.txt 2>&1; tail -3 gpurun_out/r02o_pytest.txt
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02o_smoke.txt 2>&1; tail -2 gpurun_out/r02o_smoke.txt
bash scripts/gpu_sanitize_jpeg.sh
CFGS="c3a:packed c3b:packed" TESTS=none bash scripts/gpu_ab.sh r02o
