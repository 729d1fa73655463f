"""e2e diagnosis (c2 compact path): pure host enqueue cost per call (GPU idle),
compute-only step (device arena: no DMA), DMA alone, and the pinned e2e step."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import statistics
import torch, synth
import paper_2007_13005_b200 as smol
cfg = synth.CONFIGS["c2"]
imgs, qt = synth.batch_images(cfg)
ps = smol.params_from_config(cfg)
plan = smol.Plan(ps, len(imgs))
cbs = [smol.CompactBatch(ps, imgs, qt, location="pinned") for _ in range(2)]
cbd = [smol.CompactBatch(ps, imgs, qt, location="device") for _ in range(2)]
out = plan.new_output(len(imgs))
s = torch.cuda.Stream()
res = torch.empty((1,) + tuple(out.shape[1:]), dtype=out.dtype, pin_memory=True)
def steady(batches, steps=300, d2h=True):
    for k in range(10):
        plan.run(batches[k % 2], out=out, stream=s)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for k in range(steps):
        plan.run(batches[k % 2], out=out, stream=s)
        if d2h:
            with torch.cuda.stream(s):
                res.copy_(out[:1], non_blocking=True)
    e1.record(s)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / steps
for rep in range(2):
    hts = []
    for k in range(40):
        torch.cuda.synchronize()
        t = time.perf_counter()
        plan.run(cbs[k % 2], out=out, stream=s)
        hts.append((time.perf_counter() - t) * 1e3)
    print(f"host enqueue ms/call (GPU idle): median {statistics.median(hts):.4f} min {min(hts):.4f}")
    hts = []
    for k in range(40):
        torch.cuda.synchronize()
        t = time.perf_counter()
        plan.run(cbd[k % 2], out=out, stream=s)
        hts.append((time.perf_counter() - t) * 1e3)
    print(f"host enqueue ms/call, device arena: median {statistics.median(hts):.4f}")
    print(f"compute-only (device arena) ms/step: {steady(cbd):.4f}")
    print(f"pinned e2e ms/step: {steady(cbs):.4f}   no d2h: {steady(cbs, d2h=False):.4f}")
d = torch.empty(cbs[0].arena_bytes, dtype=torch.uint8, device="cuda")
src = cbs[0].arena[:cbs[0].arena_bytes]
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(50):
    d.copy_(src, non_blocking=True)
e1.record()
torch.cuda.synchronize()
print(f"DMA alone ms: {e0.elapsed_time(e1) / 50:.4f}")
