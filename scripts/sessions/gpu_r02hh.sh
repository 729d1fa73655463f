#!/bin/bash
VARS="pf1 pf2" CFGS="c5:packed c2:dense c3a:packed c3b:packed" ROUNDS=2 bash scripts/gpu_var.sh r02hh
