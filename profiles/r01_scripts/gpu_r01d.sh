#!/bin/bash
# round-1 session d: compact transport parity + full GPU suite + bench lines (e2e via run_compact)
TAG=${1:-d}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/gpu_$TAG.txt 2>&1
timeout 600 python -m pytest tests/test_compact.py -q -p no:cacheprovider > gpurun_out/pytest_compact_$TAG.txt 2>&1
tail -3 gpurun_out/pytest_compact_$TAG.txt
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu_$TAG.txt 2>&1
tail -3 gpurun_out/pytest_gpu_$TAG.txt
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
cat gpurun_out/bench_$TAG.json
for cfg in c3a c3b c5; do
  timeout 300 python bench.py --config $cfg --layout packed --steps 500 --no-cpu-baseline > gpurun_out/cfg_${TAG}_$cfg.json 2>&1
  python -c "import json;d=json.loads(open('gpurun_out/cfg_${TAG}_$cfg.json').read().strip().splitlines()[-1]);print('$cfg', round(d['value']), round(d['roofline']['frac'],3), d['e2e'])" 2>&1 | tail -1
done
