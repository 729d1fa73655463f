#!/bin/bash
# session r: warp-per-image 1/8 kernel (thumb) -- parity + A/B on c4
TAG=${1:-r}
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu_$TAG.txt 2>&1; tail -3 gpurun_out/pytest_gpu_$TAG.txt
for r in 1 2; do for m in 0 1; do
  for lay in packed dense; do
    SMOL_THUMB=$m timeout 300 python bench.py --config c4 --layout $lay --steps 1000 --no-cpu-baseline --e2e-steps 2 > gpurun_out/thumb_${TAG}_${m}_${lay}_$r.json 2>&1
    python -c "import json;d=json.loads(open('gpurun_out/thumb_${TAG}_${m}_${lay}_$r.json').read().strip().splitlines()[-1]);print('thumb$m c4 $lay r$r', round(d['value']), round(d['roofline']['launch_ms'],4), round(d['roofline']['frac'],3))" 2>&1 | tail -1
  done
done; done
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:smol_thumb -s 5 -c 1 --csv --log-file gpurun_out/thumb_ncu_$TAG.csv python bench.py --config c4 --layout packed --steps 8 --warmup 3 --no-cpu-baseline --e2e-steps 1 > /dev/null 2>&1
grep -o '"[a-z_]*__[a-z_.]*","[^"]*","[^"]*"' gpurun_out/thumb_ncu_$TAG.csv | head -8
