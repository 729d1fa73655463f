#!/bin/bash
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "thumb or cta_config or c4" 2>&1 | tail -2
VARS="told tnew" CFGS="c4:packed" ROUNDS=3 bash scripts/gpu_var.sh r02ee
