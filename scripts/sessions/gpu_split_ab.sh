#!/bin/bash
# scale-1 split-IDCT (256 threads, 4 CTAs/SM) vs the 192-thread kernel: tests + c2 A/B
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/r02g_pytest.txt 2>&1; tail -3 gpurun_out/r02g_pytest.txt
for r in 1 2 3; do for sp in 0 1; do
  SMOL_SPLIT=$sp timeout 300 python bench.py --config c2 --steps 1000 --warmup 10 --no-cpu-baseline --e2e-steps 2 --no-eq4 --configs none > gpurun_out/q_split${sp}_$r.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/q_split${sp}_$r.json'));print('split $sp', round(d['value']), 'ms', round(d['ms_per_step'],4), 'frac', round(d['roofline']['frac'],3), d['clocks']['sm_mhz'])"
done; done
SMOL_SPLIT=1 timeout 300 ncu --set full --clock-control none --import-source on -k regex:smol_fused -c 1 -o gpurun_out/r02g_split_c2 python bench.py --config c2 --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 --no-eq4 --configs none > /dev/null 2>&1
python scripts/ncu_summary.py gpurun_out/r02g_split_c2.ncu-rep
