#!/bin/bash
TAG=${1:-t}
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu_$TAG.txt 2>&1
tail -3 gpurun_out/pytest_gpu_$TAG.txt
timeout 600 python bench.py --eq4 --no-cpu-baseline --e2e-steps 5 > gpurun_out/bench_eq4_$TAG.json 2> gpurun_out/bench_eq4_$TAG.err
tail -c 1500 gpurun_out/bench_eq4_$TAG.json
timeout 600 python bench.py --config c3a --layout packed --eq4 --no-cpu-baseline --e2e-steps 5 > gpurun_out/bench_eq4_c3a_$TAG.json 2>&1
tail -c 1200 gpurun_out/bench_eq4_c3a_$TAG.json
