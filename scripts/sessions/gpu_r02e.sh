#!/bin/bash
# round-2 re-entry baseline: GPU tests, smoke, default bench (driver command)
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/r02e_gpu.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r02e_pytest_gpu.txt 2>&1; tail -3 gpurun_out/r02e_pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r02e_smoke.txt 2>&1; tail -1 gpurun_out/r02e_smoke.txt
timeout 900 python bench.py > gpurun_out/r02e_bench.json 2> gpurun_out/r02e_bench.err; tail -c 600 gpurun_out/r02e_bench.err
python - <<'PY'
import json
d=json.load(open('gpurun_out/r02e_bench.json'))
print('c2', round(d['value']), d['roofline']['frac'], d['e2e']['value'], d['e2e'].get('pcie_frac'))
for k,v in d.get('configs',{}).items(): print(k, v)
PY
