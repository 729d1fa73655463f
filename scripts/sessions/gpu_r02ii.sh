#!/bin/bash
SMOL_LIB=build/var/lib_cp1.so timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_compact.py -m gpu -q -x -p no:cacheprovider 2>&1 | tail -1
VARS="cp0 cp1" CFGS="c2:dense c3a:packed c3b:packed c5:packed" ROUNDS=2 bash scripts/gpu_var.sh r02ii
