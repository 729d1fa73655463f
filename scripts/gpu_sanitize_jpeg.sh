#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck on the N4 JPEG kernels:
# RST index + Huffman decode inside run_jpeg (every scale / layout, samplings,
# ROI rectangles, restart intervals 0 / 1 / 5, libjpeg-written files, corrupt
# entropy data) and smol_jpeg_decode_planes
mkdir -p gpurun_out/san_jpeg
cat > /tmp/san_jpeg.py <<'PY'
import io, sys, torch, numpy as np
sys.path.insert(0, '.')
import synth, paper_2007_13005_b200 as smol
from synth import jpeg
from PIL import Image
rng = np.random.default_rng(7)
qt = synth.quant_tables(75)
files = []
for mode, ri in (("natural", 1), ("natural422", 5), ("natural444", 0), ("gray", 3), ("natural", 4)):
    files.append(jpeg.encode(synth.make_image(rng, 150, 97, qt, mode), qt, ri))
buf = io.BytesIO()
Image.fromarray(synth.natural_rgb(rng, 133, 77)).save(buf, "JPEG", quality=85, restart_marker_rows=1)
files.append(buf.getvalue())
bad = bytearray(files[0]); h = smol.jpeg_header(files[0])
bad[h["scan_offset"]:-2] = rng.bytes(len(bad) - h["scan_offset"] - 2)
files.append(bytes(bad))
planes = smol.JpegBatch(files).decode_planes()
torch.cuda.synchronize()
print("decode_planes ok", flush=True)
rects = [(10, 5, 100, 80), None, (0, 0, 150, 97), (3, 3, 40, 40), None, (20, 10, 90, 50), None]
for k in (1, 2, 4, 8):
    for lay in ("dense", "packed"):
        for idct in (("box", "truncated") if k in (2, 4) else ("box",)):
            p = smol.make_params(scale_denom=k, resize_mode="exact", resize_w=56, resize_h=48, layout=lay, idct_def=idct)
            plan = smol.Plan(p, len(files))
            for rr in (None, rects):
                for _ in range(4):          # consecutive runs through the staging slots
                    plan.run(smol.JpegBatch(files, roi_rects=rr))
            torch.cuda.synchronize()
            plan.close()
            print("run_jpeg", k, lay, idct, "ok", flush=True)
cfg = synth.CONFIGS["c2"]
imgs, qt2 = synth.distinct_images(cfg, n_distinct=4)
plan = smol.Plan(smol.params_from_config(cfg), 4)
plan.run(smol.JpegBatch([jpeg.encode(im, qt2, 1) for im in imgs])); torch.cuda.synchronize()
print("c2 ok", flush=True)
PY
for tool in memcheck racecheck synccheck; do
  timeout 1800 compute-sanitizer --tool $tool --error-exitcode 9 python /tmp/san_jpeg.py > gpurun_out/san_jpeg/sanitize_$tool.txt 2>&1
  echo "$tool rc=$?"; tail -3 gpurun_out/san_jpeg/sanitize_$tool.txt
done
