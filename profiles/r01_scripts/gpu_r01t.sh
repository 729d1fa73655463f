#!/bin/bash
# session t: torchrun path (NCCL init, max-over-ranks) at N=1, reference arm under torchrun, Eq. 4 refresh
TAG=${1:-t}
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 1 --steps 500 --warmup 5 --no-cpu-baseline > gpurun_out/torchrun_$TAG.json 2> gpurun_out/torchrun_$TAG.err; echo "torchrun rc=$?"; tail -c 400 gpurun_out/torchrun_$TAG.json
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29512 bench.py --impl reference --gpus 1 --steps 2 --warmup 3 > gpurun_out/torchrun_ref_$TAG.json 2>&1; echo "ref rc=$?"; tail -c 300 gpurun_out/torchrun_ref_$TAG.json
timeout 900 python bench.py --eq4 --steps 1000 --no-cpu-baseline > gpurun_out/eq4_$TAG.json 2> gpurun_out/eq4_$TAG.err; python -c "import json;d=json.load(open('gpurun_out/eq4_$TAG.json'));print(json.dumps(d['eq4']))"
