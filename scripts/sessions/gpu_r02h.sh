#!/bin/bash
# row-run / thumbnail output pointer walk + JPEG decoder v3: tests, configs, jpeg probe, ncu
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/r02h_pytest.txt 2>&1; tail -3 gpurun_out/r02h_pytest.txt
CFGS="c2:dense c3a:packed c3b:packed c4:packed c5:packed" TESTS=none bash scripts/gpu_ab.sh r02h
for ri in 4 1; do RI=$ri timeout 300 python scripts/jpeg_probe.py; done > gpurun_out/r02h_jpeg_probe.txt 2>&1
cat gpurun_out/r02h_jpeg_probe.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:smol_jpeg_decode -c 1 -o gpurun_out/r02h_jpeg_decode python scripts/jpeg_probe.py --ncu > /dev/null 2>&1
python scripts/ncu_summary.py gpurun_out/r02h_jpeg_decode.ncu-rep
