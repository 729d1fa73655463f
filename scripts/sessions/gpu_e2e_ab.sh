#!/bin/bash
for v in stage direct stage direct; do
  echo "== $v"; SMOL_LIB=build/var/lib_$v.so python scripts/e2e_probe.py 2>&1 | tail -2
done
