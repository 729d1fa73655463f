#!/bin/bash
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/pytest_nt.txt 2>&1
tail -2 gpurun_out/pytest_nt.txt
b1() { # nt tag config layout
  SMOL_THREADS=$1 timeout 300 python bench.py --config $3 --layout $4 --steps 400 --warmup 10 --no-cpu-baseline --e2e-steps 2 > gpurun_out/e5_$2.json 2>&1
  python -c "import json;d=json.load(open('gpurun_out/e5_$2.json'));print('$2', round(d['value']), round(d['ms_per_step'],4), d.get('clocks',{}).get('sm_mhz'))" 2>&1 | tail -1
}
for cl in "c2 dense" "c3a packed" "c3b packed" "c4 packed" "c5 packed" "c2 dense"; do set -- $cl
  b1 0 auto_$1_$2 $1 $2; b1 256 n256_$1_$2 $1 $2; done
./gpu_sanitize.sh
