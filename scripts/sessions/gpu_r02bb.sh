#!/bin/bash
for r in 1 2; do for v in i8 i4; do echo -n "$v "; SMOL_LIB=build/var/lib_$v.so RI=1 timeout 300 python scripts/jpeg_probe.py 2>&1 | grep "jpeg e2e" | tail -1; done; done
SMOL_LIB=build/var/lib_i4.so timeout 600 python -m pytest tests/test_jpeg.py -m gpu -q -x -p no:cacheprovider 2>&1 | tail -1
