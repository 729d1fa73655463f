#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_jpeg.py -m gpu -q -p no:cacheprovider 2>&1 | tail -3
RI=1 timeout 300 python scripts/jpeg_probe.py 2>&1 | grep "jpeg e2e"
RI=1 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02w_l.csv python scripts/jpeg_probe.py --ncu > /dev/null 2>&1
grep -E "jpeg_" gpurun_out/r02w_l.csv | awk -F'","' '{print substr($5,1,30), $NF}'
