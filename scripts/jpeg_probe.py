"""run_jpeg probe (c2): steady-state e2e ms/step from pinned JPEG files vs the
compact path; one pass for ncu (--ncu: 3 runs, then exit)."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth
import paper_2007_13005_b200 as smol
from synth import jpeg
name = os.environ.get("CFG", "c2")
ri = int(os.environ.get("RI", "4"))
cfg = synth.CONFIGS[name]
imgs, qt = synth.batch_images(cfg)
ps = smol.params_from_config(cfg, layout="dense" if cfg.scale_denom == 1 else "packed")
plan = smol.Plan(ps, len(imgs))
t0 = time.time()
files = jpeg.encode_batch(imgs, qt, ri)
print(f"{name} ri {ri}: encode {time.time() - t0:.1f} s, mean file {sum(map(len, files)) / len(files):.0f} B")
jbs = [smol.JpegBatch(files) for _ in range(2)]
out = plan.new_output(len(imgs))
s = torch.cuda.Stream()
if "--ncu" in sys.argv:
    for k in range(3):
        plan.run(jbs[k % 2], out=out, stream=s)
    torch.cuda.synchronize()
    sys.exit(0)
res = torch.empty((1,) + tuple(out.shape[1:]), dtype=out.dtype, pin_memory=True)
def steady(batches, steps=200):
    for k in range(10):
        plan.run(batches[k % 2], out=out, stream=s)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for k in range(steps):
        plan.run(batches[k % 2], out=out, stream=s)
        with torch.cuda.stream(s):
            res.copy_(out[:1], non_blocking=True)
    e1.record(s)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / steps
for rep in range(2):
    mj = steady(jbs)
    print(f"jpeg e2e ms/step {mj:.4f}  img/s {len(imgs) / mj * 1e3:.0f}  H2D {jbs[0].file_bytes / 1e6:.2f} MB")
cbs = [smol.CompactBatch(ps, imgs, qt, location="pinned") for _ in range(2)]
mc = steady(cbs)
print(f"compact e2e ms/step {mc:.4f}  img/s {len(imgs) / mc * 1e3:.0f}  H2D {cbs[0].arena_bytes / 1e6:.2f} MB")
