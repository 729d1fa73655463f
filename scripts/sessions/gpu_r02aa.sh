#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_compact.py tests/test_gray.py tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider 2>&1 | tail -2
timeout 300 python scripts/e2e_diag2.py 2>&1 | tail -6
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:expand -c 6 --log-file gpurun_out/r02aa_expand.csv python scripts/e2e_probe.py > /dev/null 2>&1
grep expand gpurun_out/r02aa_expand.csv | awk -F'","' '{print $NF}' | tr '\n' ' '
