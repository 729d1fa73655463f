#!/bin/bash
# session i: GPU tests, smoke, bench (c2 + all configs), reference arm, ncu launch list + full capture
TAG=${1:-g}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/gpu_$TAG.txt 2>&1
nproc >> gpurun_out/gpu_$TAG.txt; grep -m1 "model name" /proc/cpuinfo >> gpurun_out/gpu_$TAG.txt
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu_$TAG.txt 2>&1
tail -2 gpurun_out/pytest_gpu_$TAG.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.txt 2>&1; tail -1 gpurun_out/smoke_$TAG.txt
for c in c2 c3b; do timeout 300 python scripts/diag_e2e.py $c 2>&1 | tail -1; done
timeout 600 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
cat gpurun_out/bench_$TAG.json
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_$TAG.json 2>&1
for cfg in c1 c3a c3b c4 c5; do
  lay=packed; [ $cfg = c1 ] && lay=dense
  timeout 300 python bench.py --config $cfg --layout $lay --no-cpu-baseline > gpurun_out/cfg_${TAG}_$cfg.json 2>&1
  python -c "import json;d=json.loads(open('gpurun_out/cfg_${TAG}_$cfg.json').read().strip().splitlines()[-1]);print('$cfg', round(d['value']), round(d['ms_per_step'],4), round(d['roofline']['frac'],3), round(d['e2e']['value']))" 2>&1 | tail -1
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 80 --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 2 > gpurun_out/ncu_launch_$TAG.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:smol_fused -s 5 -c 1 -o gpurun_out/prof_$TAG python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu_full_$TAG.log 2>&1
timeout 900 ncu --set full --clock-control none -k regex:smol_expand -s 2 -c 1 -o gpurun_out/prof_expand_$TAG python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 3 > gpurun_out/ncu_expand_$TAG.log 2>&1
ls gpurun_out | grep $TAG
