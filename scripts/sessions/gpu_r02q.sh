#!/bin/bash
mkdir -p gpurun_out
VARS="b1 x2" CFGS="c3a:packed c3b:packed c5:packed c3a:dense" ROUNDS=2 bash scripts/gpu_var.sh r02q
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_oracle_variants.py -m gpu -q -x -p no:cacheprovider 2>&1 | tail -2
