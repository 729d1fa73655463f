#!/bin/bash
# launch-shape sweep: balanced CTA map at reduced scales, tile rows for c5 / c3b / c3a
mkdir -p gpurun_out
q() { timeout 300 python bench.py --config $1 --layout packed --steps 300 --warmup 10 --no-cpu-baseline --e2e-steps 2 --no-eq4 --configs none $3 > gpurun_out/sw.json 2>/dev/null; python -c "import json;d=json.load(open('gpurun_out/sw.json'));print('$1 $2', round(d['ms_per_step'],4), round(d['roofline']['frac'],3))"; }
for r in 1 2; do
for c in c3a c3b c5; do q $c map1; SMOL_CTA_MAP=2 q $c map2; done
for tr in 224 112 75 56 45; do q c5 tr$tr "--tile-rows $tr"; done
for tr in 112 75 56; do q c3a tr$tr "--tile-rows $tr"; q c3b tr$tr "--tile-rows $tr"; done
done
