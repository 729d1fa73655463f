#!/bin/bash
# session u: output tasks per grab at scale 1 (2 = default, 3, 4)
TAG=${1:-u}
for r in 1 2; do for g in 2 3 4; do
  SMOL_LIB=build/libsmol_g$g.so timeout 300 python bench.py --steps 1500 --no-cpu-baseline --e2e-steps 2 > gpurun_out/grab_${TAG}_${g}_$r.json 2>&1
  python -c "import json;d=json.loads(open('gpurun_out/grab_${TAG}_${g}_$r.json').read().strip().splitlines()[-1]);print('grab$g c2 r$r', round(d['value']), round(d['roofline']['launch_ms'],4))" 2>&1 | tail -1
done; done
