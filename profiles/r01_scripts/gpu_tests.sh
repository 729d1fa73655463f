#!/bin/bash
TAG=$1
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_$TAG.txt 2>&1
tail -4 gpurun_out/pytest_$TAG.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.txt 2>&1; echo smoke rc=$?; tail -2 gpurun_out/smoke_$TAG.txt
