#!/bin/bash
VARS="r8 r16 r32" CFGS="c4:packed c3b:packed c3a:packed" ROUNDS=2 bash scripts/gpu_var.sh r02t
