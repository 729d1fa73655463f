#!/bin/bash
mkdir -p gpurun_out
RI=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:smol_jpeg_decode -c 1 -o gpurun_out/r02y_dec python scripts/jpeg_probe.py --ncu > /dev/null 2>&1
ncu -i gpurun_out/r02y_dec.ncu-rep --page source --csv --print-source sass > gpurun_out/r02y_dec_sass.csv 2>/dev/null
rm -f gpurun_out/r02y_dec.ncu-rep
ls -la gpurun_out/r02y_dec_sass.csv
