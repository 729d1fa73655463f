#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r02k_pytest.txt 2>&1; tail -3 gpurun_out/r02k_pytest.txt
RI=1 timeout 300 python scripts/jpeg_probe.py > gpurun_out/r02k_jpeg_probe.txt 2>&1; cat gpurun_out/r02k_jpeg_probe.txt
RI=1 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02k_jpeg_launches.csv python scripts/jpeg_probe.py --ncu > /dev/null 2>&1
grep -E "jpeg|fused" gpurun_out/r02k_jpeg_launches.csv | awk -F'","' '{print substr($5,1,40), $NF}'
timeout 900 python bench.py > gpurun_out/r02k_bench.json 2> gpurun_out/r02k_bench.err
python - <<'PY'
import json
d=json.load(open('gpurun_out/r02k_bench.json'))
print('c2', round(d['value']), round(d['roofline']['frac'],3), d['roofline'].get('issue',{}).get('frac'), 'e2e', round(d['e2e']['value']), round(d['e2e']['pcie_frac'],3))
j=d['e2e'].get('jpeg',{}); print('jpeg', j.get('value'), j.get('ms_per_step'), j.get('pcie_frac'), j.get('error'))
for k,v in d.get('configs',{}).items(): print(k, round(v['value']), round(v['frac'],3), v.get('issue',{}).get('frac'))
print(d.get('clocks'), d.get('cpu_baseline',{}).get('value'))
PY
