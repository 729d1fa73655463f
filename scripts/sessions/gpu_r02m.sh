#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_jpeg.py -m gpu -q -x -p no:cacheprovider 2>&1 | tail -2
for r in 1 2; do for so in 0 1; do echo "sort $so"; SMOL_JPEG_SORT=$so RI=1 timeout 300 python scripts/jpeg_probe.py 2>&1 | grep "jpeg e2e" | tail -1; done; done
for so in 0 1; do SMOL_JPEG_SORT=$so RI=1 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02m_l$so.csv python scripts/jpeg_probe.py --ncu > /dev/null 2>&1
echo "sort $so"; grep -E "jpeg_" gpurun_out/r02m_l$so.csv | awk -F'","' '{print substr($5,1,30), $NF}' | tail -4; done
