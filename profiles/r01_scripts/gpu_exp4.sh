#!/bin/bash
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/pytest_ab.txt 2>&1
tail -2 gpurun_out/pytest_ab.txt
b1() { # lib tag config layout extra...
  local v=$1 tag=$2 cfg=$3 lay=$4; shift 4
  SMOL_LIB=$v timeout 300 python bench.py --config $cfg --layout $lay --steps 400 --warmup 10 --no-cpu-baseline --e2e-steps 2 "$@" > gpurun_out/e4_${tag}.json 2>&1
  python -c "import json;d=json.load(open('gpurun_out/e4_${tag}.json'));print('$tag', round(d['value']), round(d['ms_per_step'],4), d.get('clocks',{}).get('sm_mhz'))" 2>&1 | tail -1
}
for v in build/libsmol_*.so build/libsmol_cur.so; do b=$(basename $v .so); b1 $v ${b}_c2 c2 dense; done
for tr in 40 75 112; do b1 build/libsmol_cur.so cur_tr$tr c2 dense --tile-rows $tr; done
for cl in "c3a packed" "c3b packed" "c4 packed" "c5 packed"; do set -- $cl
  b1 build/libsmol_cur.so cur_$1 $1 $2; done
