#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck on small parity cases (SURVEY §4 tier 4)
cat > /tmp/san_case.py <<'PY'
import sys, torch, numpy as np
sys.path.insert(0, '.')
import synth, paper_2007_13005_b200 as smol
for name, n in (("c1", 8), ("c2", 2), ("c3b", 2), ("c4", 8)):
    cfg = synth.CONFIGS[name]
    imgs, qt = synth.distinct_images(cfg, n_distinct=n)
    plan = smol.Plan(smol.params_from_config(cfg), n)
    out = plan.run(smol.CoefBatch(imgs, qt))
    g = [smol.geometry(plan.params, im.width, im.height) for im in imgs]
    plan.debug_run(smol.CoefBatch(imgs, qt), g)
    torch.cuda.synchronize()
    print(name, "ok", float(out.float().abs().sum()))
PY
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 python /tmp/san_case.py > gpurun_out/sanitize_$tool.txt 2>&1
  echo "$tool rc=$?"; tail -3 gpurun_out/sanitize_$tool.txt
done
