#!/bin/bash
# e2e: staging-slot depth x expand stream A/B (compact path, c2) + bench e2e
mkdir -p gpurun_out
for r in 1 2; do for es in 0 1; do for n in 2 3; do echo -n "expand_stream $es "; SMOL_EXPAND_STREAM=$es SMOL_STAGE_SLOTS=$n timeout 300 python scripts/e2e_probe.py 2>&1 | grep "steps 200" ; done; done; done > gpurun_out/r02e_slots2.txt
cat gpurun_out/r02e_slots2.txt
for es in 0 1; do SMOL_EXPAND_STREAM=$es timeout 300 python bench.py --steps 300 --no-cpu-baseline --no-eq4 --configs none --e2e-steps 300 > gpurun_out/r02e_e2e_es$es.json 2>/dev/null
python -c "import json;d=json.load(open('gpurun_out/r02e_e2e_es$es.json'))['e2e'];print('es $es', d['value'], d['ms_per_step'], d['pcie_frac'])"; done
timeout 600 python -m pytest tests -m gpu -q -x -k "compact or expand or host or shard" 2>&1 | tail -2
