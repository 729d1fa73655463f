#!/bin/bash
# session j: expand kernel rework (padded lane buffers, 4 CTAs/image) + e2e diagnosis
TAG=${1:-j}
timeout 600 python -m pytest tests/test_compact.py -q -p no:cacheprovider > gpurun_out/pytest_compact_$TAG.txt 2>&1; tail -1 gpurun_out/pytest_compact_$TAG.txt
for c in c2 c3b; do timeout 300 python scripts/diag_e2e.py $c 2>&1 | tail -1; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:smol_ -c 40 --csv --log-file gpurun_out/launches_$TAG.csv python scripts/diag_e2e.py c2 > /dev/null 2>&1
python - <<'PY'
import csv,collections
rows=list(csv.reader(open('gpurun_out/launches_j.csv')))
hdr=None; agg=collections.defaultdict(list)
for r in rows:
    if 'Kernel Name' in r: hdr=r; continue
    if hdr and len(r)==len(hdr):
        d=dict(zip(hdr,r))
        if d.get('Metric Name')=='gpu__time_duration.sum': agg[d['Kernel Name'][:50]].append(float(d['Metric Value']))
for k,v in agg.items(): print(len(v), round(sum(v)/len(v),1), k)
PY
