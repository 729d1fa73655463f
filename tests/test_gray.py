"""Grayscale JPEGs (one component, subsampling 400): R = G = B
= Y.  CPU: geometry and compact records carry no chroma.  GPU: the fused
kernel, the staged and the compact paths against the oracle (which decodes
gray images by its own Y-only branch, pinned in test_oracle_pipeline.py)."""
import numpy as np
import pytest

import paper_2007_13005_b200 as smol
import synth
from tests import helpers

TOL = {"f32": 1e-4, "f16": 2e-3}


def _gray_images(cfg, n, seed=400, mode="gray"):
    qt = synth.quant_tables(cfg.quality)
    ss = np.random.SeedSequence(seed + cfg.index)
    return [synth.make_image(np.random.default_rng(s), cfg.width, cfg.height, qt, mode=mode)
            for s in ss.spawn(n)], qt


@pytest.mark.parametrize("name", ["c1", "c2", "c3a", "c4"])
def test_gray_geometry_has_no_chroma_blocks(name):
    cfg = synth.CONFIGS[name]
    p = smol.params_from_config(cfg)
    gc = smol.geometry(p, cfg.width, cfg.height)
    gg = smol.geometry(p, cfg.width, cfg.height, gray=True)
    luma = (gc["by1"][0] - gc["by0"][0] + 1) * (gc["bx1"][0] - gc["bx0"][0] + 1)
    assert gg["roi_blocks"] == luma < gc["roi_blocks"]
    for key in ("Wd", "Hd", "Wr", "Hr", "left", "top", "lx0", "lx1", "ly0", "ly1"):
        assert gg[key] == gc[key]


def test_gray_compact_record_is_luma_only():
    from tests.test_compact import read_record
    cfg = synth.CONFIGS["c2"]
    imgs, _ = _gray_images(cfg, 1)
    p = smol.params_from_config(cfg)
    E, (bx0, by0, nbx, nby), blocks = read_record(smol.compact_encode(p, imgs[0]))
    assert nby[1] == nby[2] == 0 and all(c == 0 for (c, _, _) in blocks)
    for (c, by, bx), blk in blocks.items():
        np.testing.assert_array_equal(blk, imgs[0].coef[0][by, bx])


# ------------------------------------------------------------------ GPU ----
def _check_gray(cfg, imgs, qt, layout="dense", location="device", compact=False, rois=None):
    import torch
    import oracle
    ps = smol.params_from_config(cfg, layout=layout)
    po = oracle.params_from_config(cfg)
    plan = smol.Plan(ps, len(imgs))
    if compact:
        b = smol.CompactBatch(ps, imgs, qt, rois=rois)
    else:
        b = smol.batch_for(ps, imgs, qt, location=location, rois=rois)
    out = plan.run(b)
    torch.cuda.synchronize()
    out = out.float().cpu().numpy()
    for i, im in enumerate(imgs):
        roi = None if rois is None else rois[i]
        ref = oracle.run_image(po, im, qt, roi).astype(np.float64)
        err = np.abs(out[i] - ref).max(axis=0)
        aff = helpers.affected_outputs(po, im, qt, roi)
        assert err[~aff].max(initial=0) <= TOL[cfg.out_dtype], (cfg.name, i, err[~aff].max())
        assert err.max() <= TOL[cfg.out_dtype] + 2.0 / (255 * 0.224)
    plan.close()
    return out


@pytest.mark.gpu
@pytest.mark.parametrize("name,layout", [("c1", "dense"), ("c2", "dense"), ("c3a", "packed"), ("c3b", "dense"),
                                         ("c4", "packed"), ("c5", "packed")])
def test_gray_parity(name, layout):
    cfg = synth.CONFIGS[name]
    imgs, qt = _gray_images(cfg, {"c5": 1, "c4": 8}.get(name, 3))
    _check_gray(cfg, imgs, qt, layout)


@pytest.mark.gpu
def test_gray_tie_free_bit_exact_u8_and_paths_agree():
    import torch
    cfg = synth.CONFIGS["c2"]
    imgs, qt = _gray_images(cfg, 3)
    imgs = [helpers.make_tie_free(im, qt, 1) for im in imgs]
    a = _check_gray(cfg, imgs, qt)
    b = _check_gray(cfg, imgs, qt, location="pinned")
    c = _check_gray(cfg, imgs, qt, compact=True)
    assert np.array_equal(a, b) and np.array_equal(a, c)


@pytest.mark.gpu
def test_mixed_gray_and_color_batch():
    """One batch mixing 4:2:0 and grayscale images: every image matches the
    oracle and equals its output in a single-kind batch."""
    import torch
    cfg = synth.CONFIGS["c2"]
    gray, qt = _gray_images(cfg, 3)
    color, _ = synth.distinct_images(cfg, n_distinct=3)
    mixed = [gray[0], color[0], color[1], gray[1], gray[2], color[2]]
    out = _check_gray(cfg, mixed, qt)
    ps = smol.params_from_config(cfg)
    plan = smol.Plan(ps, 3)
    og = plan.run(smol.batch_for(ps, gray, qt)).float().cpu().numpy()
    oc = plan.run(smol.batch_for(ps, color, qt)).float().cpu().numpy()
    for i, j in ((0, 0), (3, 1), (4, 2)):
        assert np.array_equal(out[i], og[j])
    for i, j in ((1, 0), (2, 1), (5, 2)):
        assert np.array_equal(out[i], oc[j])
    _check_gray(cfg, mixed, qt, compact=True)


@pytest.mark.gpu
def test_gray_poison_outside_roi():
    import torch
    cfg = synth.CONFIGS["c2"]
    imgs, qt = _gray_images(cfg, 2)
    ps = smol.params_from_config(cfg)
    plan = smol.Plan(ps, 2)
    clean = plan.run(smol.batch_for(ps, imgs, qt)).clone()
    bad = []
    for im in imgs:
        g = smol.geometry(ps, im.width, im.height, gray=True)
        c = im.coef[0].copy()
        keep = np.zeros(c.shape[:2], bool)
        keep[g["by0"][0]:g["by1"][0] + 1, g["bx0"][0]:g["bx1"][0] + 1] = True
        c[~keep] = 32767
        bad.append(synth.CoefImage(im.width, im.height, [c], (0,)))
    dirty = plan.run(smol.batch_for(ps, bad, qt))
    torch.cuda.synchronize()
    assert torch.equal(clean, dirty)
