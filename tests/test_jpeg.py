"""GPU entropy decoding of baseline JPEG (
include/smol_preproc.h "JPEG input").

CPU: the library's header reader against the oracle's (oracle/smol_oracle_jpeg.c,
pinned in test_oracle_jpeg.py) -- sizes, block grids, restart intervals, scan
offset -- and its refusals.
GPU: the Huffman decode kernels against the oracle's sequential decoder,
bit for bit (every sampling, restart intervals 0 / 1 / odd, odd sizes, q95,
libjpeg-written files); smol_preproc_run_jpeg against smol_preproc_run on the
oracle-decoded planes, bit for bit (every scale, both layouts, Definition B,
ROI rectangles, grayscale, 4:2:2 / 4:4:4, consecutive batches through the
staging slots); and against the oracle's whole pipeline within the
north_star tolerances; full c2 batch in the bench's launch configuration.
"""
import io

import numpy as np
import pytest

import oracle
import paper_2007_13005_b200 as smol
from paper_2007_13005_b200 import _native as native
import synth
from synth import jpeg

TOL = {"f32": 1e-4, "f16": 2e-3}
MODES = ("natural", "natural422", "natural444", "gray")


def _files(mode, sizes, ri, q=75, seed=0):
    qt = synth.quant_tables(q)
    rng = np.random.default_rng(seed)
    imgs = [synth.make_image(rng, w, h, qt, mode) for (w, h) in sizes]
    return imgs, qt, [jpeg.encode(im, qt, ri) for im in imgs]


# ------------------------------------------------------------------ CPU ----
@pytest.mark.parametrize("mode", MODES)
@pytest.mark.parametrize("ri", [0, 1, 5])
def test_header_matches_oracle(mode, ri):
    _, _, files = _files(mode, [(37, 29), (500, 375), (161, 161)], ri)
    for f in files:
        h = smol.jpeg_header(f)
        info = oracle.jpeg_info(f)
        assert (h["width"], h["height"], h["ncomp"], h["restart_interval"]) == \
               (info.width, info.height, info.ncomp, info.restart_interval)
        assert h["blocks_w"] == list(info.blocks_w)[:info.ncomp]
        assert h["blocks_h"] == list(info.blocks_h)[:info.ncomp]
        nmcu = info.mcus_x * info.mcus_y
        assert h["n_segments"] == (-(-nmcu // ri) if ri else 1)
        assert f[h["scan_offset"] - 14:h["scan_offset"] - 12] == b"\xff\xda" or \
               f[h["scan_offset"] - 10:h["scan_offset"] - 8] == b"\xff\xda"          # SOS just before
        assert h["subsampling"] == (400 if mode == "gray" else int(mode[-3:]) if mode != "natural" else 420)


def test_header_refusals():
    from PIL import Image
    rgb = synth.natural_rgb(np.random.default_rng(2), 40, 32)
    buf = io.BytesIO()
    Image.fromarray(rgb).save(buf, "JPEG", progressive=True)
    with pytest.raises(smol.SmolError) as e:
        smol.jpeg_header(buf.getvalue())
    assert e.value.status == native.SMOL_ERR_UNSUPPORTED
    _, _, files = _files("natural", [(40, 40)], 2)
    with pytest.raises(smol.SmolError) as e:
        smol.jpeg_header(files[0][:100])
    assert e.value.status == native.SMOL_ERR_INVALID
    with pytest.raises(smol.SmolError):
        smol.jpeg_header(b"\x00\x00" + files[0][2:])
    # 4:1:1 (luma 4x1) is not one of the supported samplings
    buf = io.BytesIO()
    Image.fromarray(rgb).save(buf, "JPEG")
    b = bytearray(buf.getvalue())
    k = bytes(b).find(b"\xff\xc0")
    b[k + 11] = 0x41
    with pytest.raises(smol.SmolError) as e:
        smol.jpeg_header(bytes(b))
    assert e.value.status == native.SMOL_ERR_UNSUPPORTED


# ------------------------------------------------------------------ GPU ----
def _oracle_planes(files):
    return [oracle.jpeg_decode(f) for f in files]


def _check_planes(files):
    jb = smol.JpegBatch(files)
    got = jb.decode_planes()
    for f, g, (info, planes, _) in zip(files, got, _oracle_planes(files)):
        assert len(g) == info.ncomp
        for c in range(info.ncomp):
            np.testing.assert_array_equal(g[c].cpu().numpy(), planes[c])


@pytest.mark.gpu
@pytest.mark.parametrize("mode", MODES)
@pytest.mark.parametrize("ri", [0, 1, 3, 7])
def test_gpu_huffman_equals_oracle(mode, ri):
    _, _, files = _files(mode, [(37, 29), (123, 77), (500, 375), (16, 16), (8, 200)], ri, seed=ri)
    _check_planes(files)


@pytest.mark.gpu
def test_gpu_huffman_q95_and_libjpeg_files():
    _, _, files = _files("natural", [(300, 200), (161, 161)], 4, q=95, seed=9)
    from PIL import Image
    rgb = synth.natural_rgb(np.random.default_rng(3), 250, 170)
    for kw in (dict(quality=90, subsampling=0, restart_marker_blocks=5),
               dict(quality=80, subsampling=1, restart_marker_rows=1),
               dict(quality=75, subsampling=2, restart_marker_blocks=1),
               dict(quality=75, subsampling=2)):
        buf = io.BytesIO()
        Image.fromarray(rgb).save(buf, "JPEG", **kw)
        files.append(buf.getvalue())
    buf = io.BytesIO()
    Image.fromarray(rgb).convert("L").save(buf, "JPEG", quality=85, restart_marker_blocks=3)
    files.append(buf.getvalue())
    _check_planes(files)


def _coef_images(files):
    """The oracle's entropy decode as CoefImages + the batch's qtables."""
    dec = _oracle_planes(files)
    qts, imgs = [], []
    for info, planes, qt in dec:
        ids = []
        for c in range(info.ncomp):
            q = qt[info.tq[c]]
            k = next((j for j, t in enumerate(qts) if np.array_equal(t, q)), None)
            if k is None:
                qts.append(q)
                k = len(qts) - 1
            ids.append(k)
        sub = 400 if info.ncomp == 1 else {(2, 2): 420, (2, 1): 422, (1, 1): 444}[(info.h[0], info.v[0])]
        imgs.append(synth.CoefImage(info.width, info.height, list(planes), tuple(ids), subsampling=sub))
    return imgs, np.stack(qts)


def _per_image(plan, params, imgs, qt, rois, roi_rects):
    """smol_preproc_run image by image, each with its own (<= 3) tables."""
    import torch
    outs = []
    for i, im in enumerate(imgs):
        ids = list(dict.fromkeys(im.qidx))
        local = synth.CoefImage(im.width, im.height, im.coef, tuple(ids.index(t) for t in im.qidx),
                                subsampling=im.subsampling)
        outs.append(plan.run(smol.batch_for(params, [local], qt[ids],
                                            rois=None if rois is None else [rois[i]],
                                            roi_rects=None if roi_rects is None else [roi_rects[i]])))
    return torch.cat(outs)


def _run_pair(params, files, rois=None, roi_rects=None):
    """(run_jpeg output, run on the oracle-decoded planes)."""
    import torch
    imgs, qt = _coef_images(files)
    plan = smol.Plan(params, len(files))
    out_j = plan.run(smol.JpegBatch(files, rois=rois, roi_rects=roi_rects))
    if len(qt) <= 4:
        out_d = plan.run(smol.batch_for(params, imgs, qt, rois=rois, roi_rects=roi_rects))
    else:
        # more distinct tables than smol_preproc_run's 4 (run_jpeg takes up
        # to 64): the reference image by image (outputs do not depend on the
        # batch -- shard invariance)
        out_d = _per_image(plan, params, imgs, qt, rois, roi_rects)
    torch.cuda.synchronize()
    r = out_j.cpu().numpy(), out_d.cpu().numpy()
    plan.close()
    return r


@pytest.mark.gpu
@pytest.mark.parametrize("name,layout", [("c1", "dense"), ("c2", "dense"), ("c3a", "packed"), ("c3b", "packed"),
                                         ("c3a", "dense"), ("c4", "packed"), ("c4", "dense")])
def test_run_jpeg_equals_run_on_decoded_planes(name, layout):
    cfg = synth.CONFIGS[name]
    imgs, qt = synth.distinct_images(cfg, n_distinct=6)
    files = [jpeg.encode(im, qt, ri) for im, ri in zip(imgs, [0, 1, 2, 3, 4, 7])]
    a, b = _run_pair(smol.params_from_config(cfg, layout=layout), files)
    np.testing.assert_array_equal(a, b)


@pytest.mark.gpu
@pytest.mark.parametrize("mode", MODES)
def test_run_jpeg_samplings_and_definition_b(mode):
    cfg = synth.CONFIGS["c3b"]
    _, _, files = _files(mode, [(500, 375), (333, 250), (161, 200)], 3, seed=5)
    for layout, idct in (("packed", "box"), ("dense", "truncated"), ("packed", "truncated")):
        a, b = _run_pair(smol.params_from_config(cfg, layout=layout, idct_def=idct), files)
        np.testing.assert_array_equal(a, b)


@pytest.mark.gpu
def test_run_jpeg_roi_rectangles_and_origins():
    cfg = synth.CONFIGS["c2"]
    _, _, files = _files("natural", [(500, 375)] * 3 + [(640, 480)], 4, seed=6)
    a, b = _run_pair(smol.params_from_config(cfg), files,
                     roi_rects=[(10, 20, 300, 200), None, (0, 0, 500, 375), (100, 50, 64, 80)])
    np.testing.assert_array_equal(a, b)
    a, b = _run_pair(smol.params_from_config(cfg), files, rois=[(0, 0), (100, 30), (-1, -1), (5, 7)])
    np.testing.assert_array_equal(a, b)


@pytest.mark.gpu
def test_run_jpeg_against_oracle_pipeline():
    import torch
    cfg = synth.CONFIGS["c2"]
    imgs, qt = synth.distinct_images(cfg, n_distinct=4)
    files = [jpeg.encode(im, qt, 4) for im in imgs]
    plan = smol.Plan(smol.params_from_config(cfg), len(files))
    out = plan.run(smol.JpegBatch(files))
    torch.cuda.synchronize()
    got = out.cpu().numpy()
    po = oracle.params_from_config(cfg)
    from tests import helpers
    for i, im in enumerate(imgs):
        ref = oracle.run_image(po, im, qt)
        err = np.abs(got[i] - ref)
        # the decoded planes equal synth's (round trip); slack only where the
        # oracle's u8 sample sits in the reading-R3 tie band
        in_band = any(bool(band.any()) for _, _, band in helpers.oracle_planes(po, im, qt))
        assert err.max() <= TOL["f32"] + (2.0 / (255 * 0.224) if in_band else 0.0)


@pytest.mark.gpu
def test_run_jpeg_consecutive_batches_through_the_slots():
    import torch
    cfg = synth.CONFIGS["c3b"]
    params = smol.params_from_config(cfg, layout="packed")
    batches = []
    for s in range(5):
        _, _, files = _files("natural", [(500, 375), (400, 300), (200, 500)], 1 + s, seed=20 + s)
        batches.append(files)
    plan = smol.Plan(params, 3)
    outs = [plan.run(smol.JpegBatch(f)) for f in batches]        # back to back, no sync
    torch.cuda.synchronize()
    for f, o in zip(batches, outs):
        imgs, qt = _coef_images(f)
        ref = plan.run(smol.batch_for(params, imgs, qt))
        torch.cuda.synchronize()
        np.testing.assert_array_equal(o.cpu().numpy(), ref.cpu().numpy())


@pytest.mark.gpu
def test_run_jpeg_full_c2_batch_sampled():
    """BASELINE c2 size (256 images, 64 distinct) in the bench's launch
    configuration; every distinct image compared with run on its planes."""
    import torch
    cfg = synth.CONFIGS["c2"]
    imgs, qt = synth.batch_images(cfg)
    files = jpeg.encode_batch(imgs, qt, 4)
    params = smol.params_from_config(cfg)
    plan = smol.Plan(params, len(files))
    out_j = plan.run(smol.JpegBatch(files))
    out_d = plan.run(smol.batch_for(params, imgs, qt))
    torch.cuda.synchronize()
    np.testing.assert_array_equal(out_j[:64].cpu().numpy(), out_d[:64].cpu().numpy())
    np.testing.assert_array_equal(out_j[-8:].cpu().numpy(), out_d[-8:].cpu().numpy())


@pytest.mark.gpu
@pytest.mark.parametrize("k,layout", [(1, "dense"), (2, "packed"), (4, "packed"), (8, "packed"), (4, "dense")])
def test_run_jpeg_corrupt_entropy_data_is_contained(k, layout):
    """Garbage in the entropy-coded data, truncated scans, stray RST markers:
    the kernels stay in bounds -- the runs succeed and a later clean run in
    the same context still matches (a fault would be sticky); only samples
    change.  (compute-sanitizer is closed on this GPU pool: this test and the
    kernels' clamps are the bounds evidence.)"""
    import torch
    rng = np.random.default_rng(k)
    _, _, files = _files("natural", [(64, 64), (97, 61), (150, 120), (40, 33)], 1 + k % 3, seed=3 + k)
    bad = []
    for i, f in enumerate(files):
        h = smol.jpeg_header(f)
        b = bytearray(f)
        body = bytearray(rng.bytes(len(f) - h["scan_offset"] - 2))
        if i == 1:                                   # stray RST markers everywhere
            for j in range(0, len(body) - 1, 7):
                body[j], body[j + 1] = 0xFF, 0xD0 + (j % 8)
        b[h["scan_offset"]:-2] = body
        if i == 2:
            b = b[:h["scan_offset"] + 5]             # truncated scan, no EOI
        bad.append(bytes(b))
    params = smol.make_params(scale_denom=k, resize_mode="exact", resize_w=48, resize_h=40, layout=layout)
    plan = smol.Plan(params, 4)
    for _ in range(3):
        plan.run(smol.JpegBatch(bad, roi_rects=[None, (5, 5, 50, 40), None, (0, 0, 40, 33)]))
    torch.cuda.synchronize()
    planes = smol.JpegBatch(bad).decode_planes()
    torch.cuda.synchronize()
    a, b = _run_pair(params, files)
    np.testing.assert_array_equal(a, b)


@pytest.mark.gpu
def test_run_jpeg_mixed_tables_in_one_batch():
    """A batch whose files carry different quantization tables (q50 / q75 / q95)
    and different Huffman tables (libjpeg's optimized per-image tables): several
    table sets, so the decoder reads its LUTs from global memory; equal to run
    on the oracle-decoded planes."""
    from PIL import Image
    rng = np.random.default_rng(12)
    files = []
    for q in (50, 75, 95):
        qt = synth.quant_tables(q)
        files.append(jpeg.encode(synth.make_image(rng, 200, 150, qt, "natural"), qt, 2))
    for opt in (True, False):
        buf = io.BytesIO()
        Image.fromarray(synth.natural_rgb(rng, 200, 150)).save(buf, "JPEG", quality=80, optimize=opt,
                                                                restart_marker_blocks=3)
        files.append(buf.getvalue())
    for name, layout in (("c3b", "packed"), ("c2", "dense")):
        a, b = _run_pair(smol.params_from_config(synth.CONFIGS[name], layout=layout), files)
        np.testing.assert_array_equal(a, b)


@pytest.mark.gpu
def test_run_jpeg_errors():
    """Batch-level refusals of smol_preproc_run_jpeg: status and message."""
    import ctypes
    import torch
    _, _, files = _files("natural", [(64, 64)] * 3, 1, seed=2)
    params = smol.params_from_config(synth.CONFIGS["c1"])
    plan = smol.Plan(params, 2)
    with pytest.raises(smol.SmolError) as e:               # more images than the plan holds
        plan.run(smol.JpegBatch(files))
    assert e.value.status == native.SMOL_ERR_CAPACITY
    bad = list(files[:2])
    bad[1] = bad[1][:2] + b"\xff\xc2" + bad[1][4:]          # image 1: progressive SOF marker first
    with pytest.raises(smol.SmolError) as e:
        plan.run(smol.JpegBatch(bad))
    assert "image 1" in str(e.value)
    jb = smol.JpegBatch(files[:2])
    jb.images[1].offset += 1                               # not 16-B aligned
    with pytest.raises(smol.SmolError) as e:
        plan.run(jb)
    assert e.value.status == native.SMOL_ERR_INVALID
    jb = smol.JpegBatch(files[:2])
    dev = jb.arena.cuda()                                  # device arena: headers cannot be parsed
    jb.desc.arena = dev.data_ptr()
    with pytest.raises(smol.SmolError) as e:
        plan.run(jb)
    assert e.value.status == native.SMOL_ERR_INVALID
    out = plan.run(smol.JpegBatch(files[:2]))              # the plan still works
    torch.cuda.synchronize()
    assert torch.isfinite(out).all()


@pytest.mark.gpu
def test_run_jpeg_large_frames():
    """Maximum sizes of the path through the JPEG input: 1080p frames (c5
    params: 1/4 scale, packed) and a 12 MP photo at 1/8 with column tiles;
    GPU entropy decode == oracle, run_jpeg == run on the decoded planes."""
    qt = synth.quant_tables(75)
    rng = np.random.default_rng(21)
    hd = [jpeg.encode(synth.make_image(rng, 1920, 1080, qt, "natural"), qt, 4)]
    _check_planes(hd)
    a, b = _run_pair(smol.params_from_config(synth.CONFIGS["c5"], layout="packed"), hd)
    np.testing.assert_array_equal(a, b)
    big = [jpeg.encode(synth.make_image(rng, 4000, 3000, qt, "natural"), qt, 8)]
    cfg = synth.Config("big8", 1, 4000, 3000, 8, "exact", resize_w=250, resize_h=188)
    a, b = _run_pair(smol.params_from_config(cfg), big)
    np.testing.assert_array_equal(a, b)
