#!/bin/bash
mkdir -p gpurun_out
for ri in 4 2 1; do RI=$ri timeout 300 python scripts/jpeg_probe.py; done > gpurun_out/r02f_jpeg_probe.txt 2>&1
cat gpurun_out/r02f_jpeg_probe.txt
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02f_jpeg_launches.csv python scripts/jpeg_probe.py --ncu > /dev/null 2>&1
grep -E "jpeg|fused" gpurun_out/r02f_jpeg_launches.csv | awk -F'","' '{print $5, $NF}' | cut -c1-150
timeout 600 ncu --set full --clock-control none --import-source on -k regex:smol_jpeg_decode -c 1 -o gpurun_out/r02f_jpeg_decode python scripts/jpeg_probe.py --ncu > /dev/null 2>&1; ls -la gpurun_out/*.ncu-rep
