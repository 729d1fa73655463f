"""Where does the compact e2e step go?  host time per call, H2D alone,
device-arena compact run (expand + fused), pinned compact run, with/without D2H."""
import sys, time, json
sys.path.insert(0, ".")
import torch
import numpy as np
import synth
import paper_2007_13005_b200 as smol

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
cfg = synth.CONFIGS[name]
lay = "dense" if name in ("c1", "c2") else "packed"
ps = smol.params_from_config(cfg, layout=lay)
imgs, qt = synth.batch_images(cfg)
plan = smol.Plan(ps, len(imgs))
out = plan.new_output(len(imgs))
stream = torch.cuda.Stream()
pin = [smol.CompactBatch(ps, imgs, qt, location="pinned") for _ in range(2)]
dev = [smol.CompactBatch(ps, imgs, qt, location="device") for _ in range(2)]
res = torch.empty((1,) + tuple(out.shape[1:]), dtype=out.dtype, pin_memory=True)
R = {}

def timed(fn, k=20):
    for i in range(3):
        fn(i)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record(stream)
    for i in range(k):
        fn(i)
    t1 = time.perf_counter()
    e1.record(stream)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / k, (t1 - t0) / k * 1e3

def run_pin(i):
    plan.run(pin[i % 2], out=out, stream=stream)

def run_pin_d2h(i):
    plan.run(pin[i % 2], out=out, stream=stream)
    with torch.cuda.stream(stream):
        res.copy_(out[:1], non_blocking=True)

def run_dev(i):
    plan.run(dev[i % 2], out=out, stream=stream)

dense = smol.batch_for(ps, imgs, qt)
def run_dense(i):
    plan.run(dense, out=out, stream=stream)

R["dense_run"] = timed(run_dense)
R["compact_device_arena"] = timed(run_dev)
R["compact_pinned"] = timed(run_pin)
R["compact_pinned_d2h"] = timed(run_pin_d2h)
# H2D alone
dst = torch.empty(pin[0].arena.numel(), dtype=torch.uint8, device="cuda")
def h2d(i):
    with torch.cuda.stream(stream):
        dst.copy_(pin[i % 2].arena, non_blocking=True)
R["h2d_only"] = timed(h2d)
R["arena_bytes"] = pin[0].arena_bytes
# host latency of one call with the GPU idle (no blocking on earlier work)
import statistics
for nm, fn in (("dense", run_dense), ("compact_dev", run_dev), ("compact_pin", run_pin)):
    ts = []
    for i in range(20):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fn(i)
        ts.append((time.perf_counter() - t0) * 1e6)
    torch.cuda.synchronize()
    R["host_us_" + nm] = statistics.median(ts)
# per-step GPU deltas of the pinned compact loop (events on the compute stream)
evs = [torch.cuda.Event(enable_timing=True) for _ in range(11)]
torch.cuda.synchronize()
evs[0].record(stream)
for i in range(10):
    run_pin(i)
    evs[i + 1].record(stream)
torch.cuda.synchronize()
R["pin_step_ms"] = [round(evs[i].elapsed_time(evs[i + 1]), 3) for i in range(10)]
print(json.dumps({name: R}))
