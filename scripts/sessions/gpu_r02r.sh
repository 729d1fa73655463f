#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_jpeg.py -m gpu -q -p no:cacheprovider 2>&1 | tail -2
for r in 1 2; do for v in j0 j1; do echo -n "$v "; SMOL_LIB=build/var/lib_$v.so RI=1 timeout 300 python scripts/jpeg_probe.py 2>&1 | grep "jpeg e2e" | tail -1; done; done
for v in j0 j1; do SMOL_LIB=build/var/lib_$v.so RI=1 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02r_$v.csv python scripts/jpeg_probe.py --ncu > /dev/null 2>&1
echo "$v"; grep -E "jpeg_decode" gpurun_out/r02r_$v.csv | awk -F'","' '{print $NF}' | tr '\n' ' '; echo; done
