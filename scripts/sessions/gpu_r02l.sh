#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_jpeg.py -m gpu -q -x -p no:cacheprovider 2>&1 | tail -2
for spt in 1 2 4 8; do echo "spt $spt"; SMOL_JPEG_SPT=$spt RI=1 timeout 300 python scripts/jpeg_probe.py 2>&1 | grep "jpeg e2e"; done
for spt in 1 2 4; do SMOL_JPEG_SPT=$spt RI=1 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02l_l$spt.csv python scripts/jpeg_probe.py --ncu > /dev/null 2>&1
echo "spt $spt"; grep -E "jpeg_decode" gpurun_out/r02l_l$spt.csv | awk -F'","' '{print substr($5,1,30), $NF}'; done
