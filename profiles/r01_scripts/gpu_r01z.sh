#!/bin/bash
# session z: thumb kernel pair taps (t2) vs t1, 4 rounds
TAG=${1:-z}
SMOL_LIB=build/libsmol_t2.so timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -k "thumb or c4 or gray" 2>&1 | tail -1
for r in 1 2 3 4; do for v in t1 t2; do
  SMOL_LIB=build/libsmol_$v.so timeout 300 python bench.py --config c4 --layout packed --steps 3000 --no-cpu-baseline --e2e-steps 2 > gpurun_out/th_${TAG}_${v}_$r.json 2>&1
  python -c "import json;d=json.loads(open('gpurun_out/th_${TAG}_${v}_$r.json').read().strip().splitlines()[-1]);print('$v c4 r$r', round(d['value']), round(d['roofline']['launch_ms'],4))" 2>&1 | tail -1
done; done
