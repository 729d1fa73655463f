#!/bin/bash
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "run_host" > gpurun_out/pytest_e2e.txt 2>&1; tail -2 gpurun_out/pytest_e2e.txt
python - <<'PY'
import torch, time
a = torch.empty(256 << 20, dtype=torch.uint8).pin_memory(); d = torch.empty_like(a, device='cuda')
for _ in range(3): d.copy_(a, non_blocking=True)
torch.cuda.synchronize(); t=time.time()
for _ in range(10): d.copy_(a, non_blocking=True)
torch.cuda.synchronize(); print("H2D GB/s", 10*a.numel()/(time.time()-t)/1e9)
PY
for cl in "c2 dense" "c5 packed" "c3b packed"; do set -- $cl
timeout 300 python bench.py --config $1 --layout $2 --steps 200 --warmup 10 --no-cpu-baseline --e2e-steps 20 > gpurun_out/e2e_$1.json 2>&1
python -c "import json;d=json.load(open('gpurun_out/e2e_$1.json'));print('$1', round(d['value']), 'e2e', round(d['e2e']['value']), d['e2e']['h2d_bytes_per_step'])" 2>&1 | tail -1
done
