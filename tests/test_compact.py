"""Compact coefficient transport (include/smol_preproc.h).

CPU: the C encoder (smol_compact_encode, host only) against an independent
Python reader of the record format written from the header's description:
the record must hold exactly the ROI blocks smol_debug_geometry reports and,
per block, exactly the nonzero coefficients the scale uses (reading R1), so
decoding it gives back the input on the used set and zero elsewhere.

GPU: smol_preproc_run_compact must be bit-identical to smol_preproc_run on the
dense device planes (the compact path only changes transport), and within
the north_star tolerance of the oracle."""
import struct

import numpy as np
import pytest

import paper_2007_13005_b200 as smol
import synth
from paper_2007_13005_b200 import layout as lay

MAGIC = 0x32434D53


def read_record(rec: np.ndarray):
    """Parse one record (format: include/smol_preproc.h) ->
    (E, ranges, {(c, by, bx): int16[E] block})."""
    b = rec.tobytes()
    magic, E, nunits, zero = struct.unpack_from("<4I", b, 0)
    assert magic == MAGIC and zero == 0
    f = struct.unpack_from("<12i", b, 16)
    bx0, by0, nbx, nby = f[0:3], f[3:6], f[6:9], f[9:12]
    nblocks = sum(nbx[c] * nby[c] for c in range(3))
    nrows = sum(nby)
    lens = np.frombuffer(b, np.uint8, nblocks, 64)
    rso = -(-(64 + nblocks) // 4) * 4
    rs = np.frombuffer(b, np.uint32, nrows, rso)
    uoff = -(-(rso + 4 * nrows) // 16) * 16
    units = np.frombuffer(b, np.uint16, nunits, uoff)
    assert len(b) == -(-(uoff + 2 * nunits + 2) // 16) * 16
    blocks = {}
    k = bi = ri = 0
    for c in range(3):
        for r in range(nby[c]):
            assert rs[ri] == k               # row starts index the entry stream
            ri += 1
            for x in range(nbx[c]):
                end = k + int(lens[bi]); bi += 1
                blk = np.zeros(E, np.int16)
                last = -1
                while k < end:
                    u = int(units[k]); k += 1
                    pos, v = u & 63, (u >> 6) - (1024 if u >> 15 else 0)
                    if v == -512:
                        v = int(np.int16(units[k])); k += 1
                        assert not -511 <= v <= 511      # escapes only for large values
                    assert v != 0 and pos > last and pos < E
                    last = pos
                    blk[pos] = v
                blocks[(c, by0[c] + r, bx0[c] + x)] = blk
    assert k == nunits
    return E, (bx0, by0, nbx, nby), blocks


def used_elements(k: int, packed: bool):
    """Element indices of a stored block that scale 1/k uses (reading R1),
    from the layout's index sets (not from the C mask)."""
    idx = lay.index_set(k)
    return list(range(len(idx))) if (packed and k > 1) else idx


@pytest.mark.parametrize("name,layout,quality", [("c1", "dense", 75), ("c2", "dense", 75), ("c2", "dense", 95),
                                                 ("c3a", "dense", 75), ("c3a", "packed", 75),
                                                 ("c3b", "packed", 95), ("c4", "packed", 75),
                                                 ("c4", "dense", 75)])
def test_encoder_roundtrip_against_python_reader(name, layout, quality):
    cfg = synth.CONFIGS[name]
    imgs, _ = synth.distinct_images(cfg, n_distinct=2, quality=quality)
    p = smol.params_from_config(cfg, layout=layout)
    k = cfg.scale_denom
    packed = layout == "packed"
    used = used_elements(k, packed)
    for im in imgs:
        rec = smol.compact_encode(p, im)
        assert rec.size % 16 == 0
        E, (bx0, by0, nbx, nby), blocks = read_record(rec)
        assert E == lay.block_elems(k, packed)
        g = smol.geometry(p, im.width, im.height)
        for c in range(3):
            assert (bx0[c], by0[c]) == (g["bx0"][c], g["by0"][c])
            assert (bx0[c] + nbx[c] - 1, by0[c] + nby[c] - 1) == (g["bx1"][c], g["by1"][c])
        assert len(blocks) == g["roi_blocks"]
        stored = [lay.pack_plane(np.asarray(cc, np.int16), k if packed else 1) for cc in im.coef]
        for (c, by, bx), blk in blocks.items():
            src = stored[c][by, bx * E:(bx + 1) * E]
            want = np.zeros(E, np.int16)
            want[used] = src[used]
            np.testing.assert_array_equal(blk, want, err_msg=f"{name} comp {c} block ({by},{bx})")


def test_encoder_roundtrip_stress_escapes():
    """Dense uniform coefficients with small quantisers: many |v| > 511 (escape
    entries) and odd sizes."""
    rng = np.random.default_rng(13005)
    qt = synth.quant_tables(95)
    p = smol.params_from_config(synth.CONFIGS["c2"], resize_short=64, crop_w=48, crop_h=40)
    n_esc = 0
    for (w, h) in [(97, 61), (200, 333), (64, 64)]:
        im = synth.make_image(rng, w, h, qt, mode="stress")
        E, _, blocks = read_record(smol.compact_encode(p, im))
        for (c, by, bx), blk in blocks.items():
            np.testing.assert_array_equal(blk, np.asarray(im.coef[c][by, bx], np.int16))
            n_esc += int((np.abs(blk.astype(np.int32)) > 511).sum())
    assert n_esc > 100


def test_encoder_size_query_capacity_and_compression():
    cfg = synth.CONFIGS["c2"]
    imgs, _ = synth.distinct_images(cfg, n_distinct=2)
    p = smol.params_from_config(cfg)
    im = imgs[0]
    rec = smol.compact_encode(p, im)
    planes = [lay.pack_plane(np.asarray(c, np.int16), 1) for c in im.coef]
    d = smol._desc_for(im.width, im.height, [c.shape[1] for c in im.coef], [c.shape[0] for c in im.coef],
                       tuple(im.qidx), None, strides=[2 * q.shape[1] for q in planes])
    import ctypes
    for ci in range(3):
        d.coef[ci] = planes[ci].ctypes.data
    n = ctypes.c_int64()
    smol.check(smol.lib().smol_compact_encode(ctypes.byref(p), ctypes.byref(d), None, 0, ctypes.byref(n)))
    assert n.value == rec.size
    small = np.zeros(rec.size - 16, np.uint8)
    rc = smol.lib().smol_compact_encode(ctypes.byref(p), ctypes.byref(d), small.ctypes.data, small.size,
                                        ctypes.byref(n))
    assert rc == 5                                    # SMOL_ERR_CAPACITY
    # natural q75 coefficients: far fewer bytes than the dense ROI blocks
    g = smol.geometry(p, im.width, im.height)
    assert rec.size < 0.25 * g["roi_coef_bytes"], (rec.size, g["roi_coef_bytes"])
    # an all-zero image: header + bitmaps + row starts only
    z = synth.CoefImage(im.width, im.height, [np.zeros_like(c) for c in im.coef])
    _, _, blocks = read_record(smol.compact_encode(p, z))
    assert all(not b.any() for b in blocks.values())


def test_encoder_explicit_roi_and_errors():
    cfg = synth.CONFIGS["c2"]
    imgs, _ = synth.distinct_images(cfg, n_distinct=1)
    p = smol.params_from_config(cfg)
    im = imgs[0]
    g = smol.geometry(p, im.width, im.height, roi=(0, 0))
    _, (bx0, by0, nbx, nby), _ = read_record(smol.compact_encode(p, im, roi=(0, 0)))
    assert (bx0[0], by0[0]) == (g["bx0"][0], g["by0"][0]) == (0, 0)
    with pytest.raises(smol.SmolError) as e:
        smol.compact_encode(p, im, roi=(500, 0))       # outside the resized image
    assert e.value.status == 1


# ------------------------------------------------------------------ GPU ----
@pytest.mark.gpu
@pytest.mark.parametrize("name,layout", [("c1", "dense"), ("c2", "dense"), ("c3a", "packed"), ("c3a", "dense"),
                                         ("c3b", "packed"), ("c4", "packed"), ("c4", "dense"), ("c5", "packed")])
def test_run_compact_equals_device(name, layout):
    import torch
    cfg = synth.CONFIGS[name]
    n = {"c5": 2, "c4": 16}.get(name, 6)
    imgs, qt = synth.distinct_images(cfg, n_distinct=n)
    ps = smol.params_from_config(cfg, layout=layout)
    plan = smol.Plan(ps, n)
    a = plan.run(smol.batch_for(ps, imgs, qt)).clone()
    cbs = [smol.CompactBatch(ps, imgs, qt, location="pinned") for _ in range(2)]
    outs = [plan.run(cbs[k % 2]).clone() for k in range(5)]       # back-to-back: double buffer
    outs.append(plan.run(smol.CompactBatch(ps, imgs, qt, location="device")))
    torch.cuda.synchronize()
    for o in outs:
        assert torch.equal(a, o), name
    plan.close()


@pytest.mark.gpu
def test_run_compact_stress_rois_and_hetero_sizes():
    import torch
    import oracle
    rng = np.random.default_rng(2007)
    cfg = synth.CONFIGS["c2"]
    qt = synth.quant_tables(95)
    imgs = [synth.make_image(rng, int(w), int(h), qt, mode=m)
            for (w, h), m in zip(synth.random_sizes(rng, 6, 40, 400), ["natural", "stress"] * 3)]
    ps = smol.params_from_config(cfg, resize_short=64, crop_w=48, crop_h=40)
    plan = smol.Plan(ps, len(imgs))
    rois = [None] * len(imgs)
    rois[1] = (0, 0)
    a = plan.run(smol.CoefBatch(imgs, qt, rois=[r if r else (-1, -1) for r in rois])).clone()
    b = plan.run(smol.CompactBatch(ps, imgs, qt, rois=[r if r else (-1, -1) for r in rois]))
    torch.cuda.synchronize()
    assert torch.equal(a, b)


@pytest.mark.gpu
def test_run_compact_rejects_foreign_records():
    cfg = synth.CONFIGS["c3a"]
    imgs, qt = synth.distinct_images(cfg, n_distinct=2)
    pd = smol.params_from_config(cfg)
    pp = smol.params_from_config(cfg, layout="packed")
    plan = smol.Plan(pp, 2)
    with pytest.raises(smol.SmolError) as e:
        plan.run(smol.CompactBatch(pd, imgs, qt))       # encoded for the dense layout
    assert e.value.status == 1 and "image 0" in str(e.value)
    cb = smol.CompactBatch(pp, imgs, qt)
    cb.desc.arena_bytes = 64
    with pytest.raises(smol.SmolError) as e:
        plan.run(cb)
    assert e.value.status == 1


def test_encoder_roundtrip_int16_extremes():
    """Full int16 range (the ABI accepts any coefficient): the escape
    boundaries -512/-511/511/512 and -32768/32767 survive the record."""
    rng = np.random.default_rng(2)
    w, h = 48, 40
    special = np.array([-32768, 32767, -512, -511, 511, 512, -1, 1, 0, 0, 0, 0], np.int16)
    coef = []
    for (bh, bw) in [(5, 6), (3, 3), (3, 3)]:
        c = rng.choice(special, size=(bh, bw, 64)).astype(np.int16)
        c[0, 0] = rng.integers(-32768, 32768, size=64, dtype=np.int64).astype(np.int16)
        coef.append(c)
    im = synth.CoefImage(w, h, coef)
    p = smol.make_params(scale_denom=1, resize_mode="exact", resize_w=w, resize_h=h)
    E, _, blocks = read_record(smol.compact_encode(p, im))
    g = smol.geometry(p, w, h)
    assert len(blocks) == g["roi_blocks"]
    for (c, by, bx), blk in blocks.items():
        np.testing.assert_array_equal(blk, coef[c][by, bx])


@pytest.mark.gpu
def test_run_compact_int16_extremes_equal_dense():
    import torch
    rng = np.random.default_rng(3)
    special = np.array([-32768, 32767, -512, -511, 511, 512, -1, 1, 0, 0, 0, 0], np.int16)
    imgs = []
    for (w, h) in [(48, 40), (130, 77)]:
        shapes = [(-(-h // 8), -(-w // 8)), (-(-h // 16), -(-w // 16)), (-(-h // 16), -(-w // 16))]
        imgs.append(synth.CoefImage(w, h, [rng.choice(special, size=s + (64,)).astype(np.int16) for s in shapes]))
    qt = synth.quant_tables(50)
    for k in (1, 2, 4):
        p = smol.params_from_config(synth.CONFIGS["c1"], scale_denom=k, resize_w=24, resize_h=16)
        plan = smol.Plan(p, len(imgs))
        a = plan.run(smol.batch_for(p, imgs, qt)).clone()
        b = plan.run(smol.CompactBatch(p, imgs, qt))
        torch.cuda.synchronize()
        assert torch.equal(a, b), k
        assert torch.isfinite(a).all()
        plan.close()


@pytest.mark.gpu
def test_run_compact_corrupt_lengths_do_not_fault():
    """Block lengths and row starts of a record are clamped inside the expand
    kernel (not re-scanned on the host): a record with lengths of 255 and
    row starts past its end gives garbage samples for that image but no
    out-of-bounds access -- the context stays usable and the other images
    of the batch are unaffected."""
    import torch
    cfg = synth.CONFIGS["c2"]
    imgs, qt = synth.distinct_images(cfg, n_distinct=3)
    ps = smol.params_from_config(cfg)
    plan = smol.Plan(ps, 3)
    good = plan.run(smol.CompactBatch(ps, imgs, qt))
    cb = smol.CompactBatch(ps, imgs, qt)
    rec0 = cb.arena.numpy()                  # pinned host arena (a view)
    g = smol.geometry(ps, imgs[0].width, imgs[0].height)
    nblocks = sum((g["bx1"][c] - g["bx0"][c] + 1) * (g["by1"][c] - g["by0"][c] + 1) for c in range(3))
    rec0[64:64 + nblocks] = 255              # image 0: every block length 255
    rs = (64 + nblocks + 3) & ~3
    rec0[rs:rs + 40] = 0xff                  # first row starts far past the record
    bad = plan.run(cb)
    torch.cuda.synchronize()                 # raises if the expand kernel faulted
    assert torch.equal(bad[1:], good[1:])
    again = plan.run(smol.CompactBatch(ps, imgs, qt))
    torch.cuda.synchronize()
    assert torch.equal(again, good)
    plan.close()
