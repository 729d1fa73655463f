#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck on the current kernels: tiled (all scales,
# CTA map, gray), expand (compact records), thumb (1/8 packed), gather (run_host)
mkdir -p gpurun_out/san2
cat > /tmp/san_case2.py <<'PY'
import sys, torch, numpy as np
sys.path.insert(0, '.')
import synth, paper_2007_13005_b200 as smol
rng = np.random.default_rng(5)
for name, n, lay in (("c1", 8, "dense"), ("c2", 3, "dense"), ("c3a", 2, "packed"), ("c3b", 2, "packed"),
                     ("c4", 8, "packed"), ("c4", 4, "dense"), ("c5", 1, "packed")):
    cfg = synth.CONFIGS[name]
    imgs, qt = synth.distinct_images(cfg, n_distinct=n)
    imgs = imgs + [synth.make_image(rng, cfg.width, cfg.height, qt, mode="gray")]
    p = smol.params_from_config(cfg, layout=lay)
    plan = smol.Plan(p, len(imgs))
    a = plan.run(smol.batch_for(p, imgs, qt)).clone()
    b = plan.run(smol.CompactBatch(p, imgs, qt)).clone()
    c = plan.run(smol.batch_for(p, imgs, qt, location="pinned")).clone()
    torch.cuda.synchronize()
    print(name, lay, "ok", torch.equal(a, b), torch.equal(a, c))
PY
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --error-exitcode 9 python /tmp/san_case2.py > gpurun_out/san2/sanitize_$tool.txt 2>&1
  echo "$tool rc=$?"; tail -4 gpurun_out/san2/sanitize_$tool.txt
done
