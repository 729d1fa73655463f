#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r02u_pytest.txt 2>&1; tail -2 gpurun_out/r02u_pytest.txt
CFGS="c3a:packed c3b:packed c5:packed c2:dense" TESTS=none bash scripts/gpu_ab.sh r02u
