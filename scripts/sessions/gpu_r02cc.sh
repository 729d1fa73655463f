#!/bin/bash
for r in 1 2; do for v in d128 d64n d64; do echo -n "$v "; SMOL_LIB=build/var/lib_$v.so RI=1 timeout 300 python scripts/jpeg_probe.py 2>&1 | grep "jpeg e2e" | tail -1; done; done
