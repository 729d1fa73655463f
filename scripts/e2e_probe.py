"""e2e probe: host time per run_compact call, device step time, H2D of the arena alone."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth
import paper_2007_13005_b200 as smol
cfg = synth.CONFIGS["c2"]
imgs, qt = synth.batch_images(cfg)
ps = smol.params_from_config(cfg)
plan = smol.Plan(ps, len(imgs))
cbs = [smol.CompactBatch(ps, imgs, qt, location="pinned") for _ in range(2)]
out = plan.new_output(len(imgs))
s = torch.cuda.Stream()
res = torch.empty((1,) + tuple(out.shape[1:]), dtype=out.dtype, pin_memory=True)
for k in range(10):
    plan.run(cbs[k % 2], out=out, stream=s)
torch.cuda.synchronize()
for steps in (50, 200):
    t0 = time.perf_counter()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    ht = 0.0
    for k in range(steps):
        a = time.perf_counter()
        plan.run(cbs[k % 2], out=out, stream=s)
        with torch.cuda.stream(s):
            res.copy_(out[:1], non_blocking=True)
        ht += time.perf_counter() - a
    e1.record(s)
    torch.cuda.synchronize()
    dev = e0.elapsed_time(e1) / steps
    print(f"slots {os.environ.get('SMOL_STAGE_SLOTS', '3')} steps {steps}: device ms/step {dev:.4f}  host ms/call {1e3 * ht / steps:.4f}  wall ms/step {1e3 * (time.perf_counter() - t0) / steps:.4f}  img/s {256 / dev * 1e3:.0f}")
# H2D of the arena alone
d = torch.empty(cbs[0].arena_bytes, dtype=torch.uint8, device="cuda")
src = cbs[0].arena[:cbs[0].arena_bytes]
for _ in range(3):
    d.copy_(src, non_blocking=True)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20):
    d.copy_(src, non_blocking=True)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 20
print(f"H2D {cbs[0].arena_bytes / 1e6:.2f} MB: {ms:.4f} ms = {cbs[0].arena_bytes / ms / 1e6:.1f} GB/s")
