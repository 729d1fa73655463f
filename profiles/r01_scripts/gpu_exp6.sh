#!/bin/bash
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/pytest_e6.txt 2>&1
tail -2 gpurun_out/pytest_e6.txt
b1() { # lib tag config layout [extra]
  local lib=$1 tag=$2 cfg=$3 lay=$4; shift 4
  SMOL_LIB=$lib timeout 300 python bench.py --config $cfg --layout $lay --steps 400 --warmup 10 --no-cpu-baseline --e2e-steps 2 "$@" > gpurun_out/e6_$tag.json 2>&1
  python -c "import json;d=json.load(open('gpurun_out/e6_$tag.json'));print('$tag', round(d['value']), round(d['ms_per_step'],4), d.get('clocks',{}).get('sm_mhz'))" 2>&1 | tail -1
}
for v in prev cur prev cur; do b1 build/libsmol_$v.so ${v}_c2 c2 dense; done
for v in prev cur; do for c in c3a c3b c4 c5; do b1 build/libsmol_$v.so ${v}_$c $c packed; done; done
