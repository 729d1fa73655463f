#!/bin/bash
TAG=$1
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/pytest_$TAG.txt 2>&1
tail -3 gpurun_out/pytest_$TAG.txt
for v in build/libsmol_*.so; do
  b=$(basename $v .so)
  SMOL_LIB=$v timeout 300 python bench.py --steps 200 --warmup 10 --no-cpu-baseline --e2e-steps 5 > gpurun_out/bench_${TAG}_$b.json 2>&1
  echo $b; python -c "import json;d=json.load(open('gpurun_out/bench_${TAG}_$b.json'));print(d['value'], d['ms_per_step'], d['roofline']['frac'])"
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:smol_ -s 5 -c 1 -o gpurun_out/prof_$TAG python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu_full_$TAG.log 2>&1
