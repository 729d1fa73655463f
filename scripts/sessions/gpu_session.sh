#!/bin/bash
# one measurement session: driver-style bench (+ reference arm, torchrun N=1),
# smoke, ncu launch list of the bench command, ncu --set full of the top
# kernel per config (+ SASS source CSV), DRAM bytes per config
TAG=${1:-s}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/gpu_$TAG.txt 2>&1
nproc >> gpurun_out/gpu_$TAG.txt; grep -m1 "model name" /proc/cpuinfo >> gpurun_out/gpu_$TAG.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.txt 2>&1; tail -1 gpurun_out/smoke_$TAG.txt
( time timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err ) 2> gpurun_out/bench_time_$TAG.txt; tail -3 gpurun_out/bench_time_$TAG.txt
python -c "
import json;d=json.loads(open('gpurun_out/bench_$TAG.json').read().strip().splitlines()[-1])
print('c2', round(d['value']), d['ms_per_step'], d['roofline']['frac'], 'e2e', round(d['e2e']['value']), 'pcie', round(d['e2e'].get('pcie_frac',0),3))
for k,v in d.get('configs',{}).items(): print(k, round(v['value']), round(v['launch_ms'],4), round(v['frac'],3))
print('eq4', {k: d.get('eq4',{}).get(k) for k in ('t_exec','pipelined_measured')}, 'cpu', d.get('cpu_baseline',{}).get('value'))
print('clocks', d.get('clocks'))"
timeout 600 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/bench_ref_$TAG.json 2>&1; tail -c 400 gpurun_out/bench_ref_$TAG.json; echo
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 1 --steps 20 --warmup 5 --configs none --no-eq4 --no-cpu-baseline > gpurun_out/bench_torchrun_$TAG.json 2>&1; tail -c 300 gpurun_out/bench_torchrun_$TAG.json; echo
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --gpus 1 --steps 20 --warmup 5 --configs none --no-eq4 --no-cpu-baseline --e2e-steps 2 > gpurun_out/ncu_launch_$TAG.log 2>&1
bash scripts/gpu_prof2.sh $TAG "c2:dense:smol_fused c3a:packed:smol_fused c3b:packed:smol_fused c4:packed:smol_thumb c5:packed:smol_fused"
ls gpurun_out | grep $TAG | wc -l
