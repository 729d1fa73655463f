#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck on the round-2 kernels:
# tiled (all scales, CTA map, gray, row runs), generic chroma (4:2:2/4:4:4),
# Definition B, chroma at twice the scale, ROI rectangles, expand (compact
# records read in place), thumbnail (row runs), gather (run_host)
mkdir -p gpurun_out/san3
cat > /tmp/san_case3.py <<'PY'
import sys, torch, numpy as np
sys.path.insert(0, '.')
import synth, paper_2007_13005_b200 as smol
rng = np.random.default_rng(5)
def run(p, imgs, qt, rects=None, tag=""):
    plan = smol.Plan(p, len(imgs))
    a = plan.run(smol.batch_for(p, imgs, qt, roi_rects=rects)).clone()
    c = plan.run(smol.batch_for(p, imgs, qt, location="pinned", roi_rects=rects)).clone()
    ok = [torch.equal(a, c)]
    if p.scale_denom != 8 or p.layout == 0:
        b = plan.run(smol.CompactBatch(p, imgs, qt, roi_rects=rects)).clone()
        ok.append(torch.equal(a, b))
    torch.cuda.synchronize()
    print(tag, "ok", ok, flush=True)
    plan.close()
for name, n, lay in (("c1", 8, "dense"), ("c2", 3, "dense"), ("c3a", 2, "packed"), ("c3b", 2, "packed"),
                     ("c4", 8, "packed"), ("c5", 1, "packed")):
    cfg = synth.CONFIGS[name]
    imgs, qt = synth.distinct_images(cfg, n_distinct=n)
    imgs = imgs + [synth.make_image(rng, cfg.width, cfg.height, qt, mode="gray")]
    run(smol.params_from_config(cfg, layout=lay), imgs, qt, tag=name)
qt = synth.quant_tables(75)
mixed = [synth.make_image(rng, 160, 120, qt, "natural444"), synth.make_image(rng, 97, 61, qt, "natural422"),
         synth.make_image(rng, 128, 96, qt), synth.make_image(rng, 64, 48, qt, "gray")]
rects = [(10, 5, 100, 90), (0, 0, 97, 61), (33, 17, 60, 40), (1, 1, 20, 20)]
for k in (1, 2, 4, 8):
    run(smol.make_params(scale_denom=k, resize_mode="exact", resize_w=56, resize_h=48, layout="packed"),
        mixed, qt, rects, tag=f"gc k={k}")
for k in (2, 4):
    run(smol.make_params(scale_denom=k, resize_mode="exact", resize_w=56, resize_h=48, idct_def="truncated",
                         layout="packed"), mixed, qt, tag=f"defB k={k}")
    cfg = synth.CONFIGS["c3a" if k == 2 else "c3b"]
    imgs, qt2 = synth.distinct_images(cfg, n_distinct=2)
    run(smol.params_from_config(cfg, chroma_2s=True), imgs, qt2, tag=f"c2s k={k}")
PY
for tool in memcheck racecheck synccheck; do
  timeout 1800 compute-sanitizer --tool $tool --error-exitcode 9 python /tmp/san_case3.py > gpurun_out/san3/sanitize_$tool.txt 2>&1
  echo "$tool rc=$?"; tail -3 gpurun_out/san3/sanitize_$tool.txt
done
