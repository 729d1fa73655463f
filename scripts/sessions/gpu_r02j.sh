#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/r02j_pytest.txt 2>&1; tail -3 gpurun_out/r02j_pytest.txt
VARS="base nrm nrmt0" CFGS="c3a:packed c3b:packed c4:packed c5:packed" ROUNDS=2 bash scripts/gpu_var.sh r02j
