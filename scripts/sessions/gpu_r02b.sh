#!/bin/bash
# new bench default run + shard test + ncu captures of the current kernels
TAG=${1:-r02b}
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_shard_gpu.py -q -p no:cacheprovider > gpurun_out/pytest_shard_$TAG.txt 2>&1; tail -2 gpurun_out/pytest_shard_$TAG.txt
/usr/bin/time -v timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; grep -E "Elapsed" gpurun_out/bench_$TAG.err; tail -c 3000 gpurun_out/bench_$TAG.json
bash scripts/gpu_prof2.sh $TAG
