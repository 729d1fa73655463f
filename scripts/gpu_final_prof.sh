#!/bin/bash
# final round-2 evidence: ncu --set full of each config's main kernel (bench
# launch configuration), the JPEG kernels, and the launch list of the default
# bench command; summaries + traffic.json update
TAG=${1:-r02z}
mkdir -p gpurun_out/$TAG
for cl in c2:dense:smol_fused c3a:packed:smol_fused c3b:packed:smol_fused c4:packed:smol_thumb c5:packed:smol_fused; do
  IFS=: read cfg lay k <<< "$cl"
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -c 1 -o gpurun_out/$TAG/ncu_$cfg \
    python bench.py --config $cfg --layout $lay --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 --no-eq4 --configs none > /dev/null 2>&1
  python scripts/ncu_summary.py gpurun_out/$TAG/ncu_$cfg.ncu-rep > gpurun_out/$TAG/ncu_${cfg}_summary.txt 2>&1
  head -4 gpurun_out/$TAG/ncu_${cfg}_summary.txt
  rm -f gpurun_out/$TAG/ncu_$cfg.ncu-rep        # (gpurun copies back <= 64 MiB)
done
for k in smol_jpeg_decode smol_jpeg_index; do
  RI=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -c 1 -o gpurun_out/$TAG/ncu_$k python scripts/jpeg_probe.py --ncu > /dev/null 2>&1
  python scripts/ncu_summary.py gpurun_out/$TAG/ncu_$k.ncu-rep > gpurun_out/$TAG/ncu_${k}_summary.txt 2>&1
  head -3 gpurun_out/$TAG/ncu_${k}_summary.txt
  rm -f gpurun_out/$TAG/ncu_$k.ncu-rep
done
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/$TAG/launches_default_bench.csv \
  python bench.py --steps 20 --warmup 3 --e2e-steps 5 > gpurun_out/$TAG/ncu_bench.log 2>&1
grep -c "smol_" gpurun_out/$TAG/launches_default_bench.csv
