#!/bin/bash
# round-2 baseline: GPU tests + quick per-config bench of the current kernels
TAG=${1:-base}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/gpu_$TAG.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu_$TAG.txt 2>&1; tail -2 gpurun_out/pytest_gpu_$TAG.txt
for cl in "c2 dense" "c3a packed" "c3b packed" "c4 packed" "c5 packed"; do
  set -- $cl
  timeout 300 python bench.py --config $1 --layout $2 --steps 300 --warmup 10 --no-cpu-baseline --e2e-steps 20 > gpurun_out/q_${TAG}_$1_$2.json 2>&1
  python -c "import json;d=json.load(open('gpurun_out/q_${TAG}_$1_$2.json'));print('$1 $2', round(d['value']), round(d['ms_per_step'],4), round(d['roofline']['launch_ms'],4), round(d['roofline']['frac'],3), round(d['e2e']['value']), d.get('clocks'))" 2>&1 | tail -1
done
