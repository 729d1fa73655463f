"""Pins of the oracle's baseline-JPEG entropy decoder (oracle/smol_oracle_jpeg.c,
ITU-T T.81 Annexes B, C, F.2.2) against things other than
itself:
  * an independent encoder (synth/jpeg.py, T.81 F.1.2): encode known
    coefficient planes, decode, exact equality -- every sampling, restart
    intervals of 0 / 1 / odd MCU counts, odd image sizes;
  * libjpeg (Pillow): files written by libjpeg's own encoder (its FDCT,
    quantizer, Huffman coder, restart markers) are decoded by the oracle, and
    the plain IDCT of the decoded coefficients (scipy idctn, level shift,
    round) matches libjpeg's decoded samples within its integer IDCT's +-1;
    libjpeg also decodes synth's files to within +-1 of the same IDCT.
"""
import io

import numpy as np
import pytest

import oracle
import synth
from synth import jpeg

SAMPLINGS = ("natural", "natural422", "natural444", "gray")


def _idct_planes(planes, qt, tq):
    from scipy import fft
    out = []
    for c, p in enumerate(planes):
        bh, bw, _ = p.shape
        d = p.astype(np.float64) * qt[tq[c]].astype(np.float64)
        v = fft.idctn(d.reshape(bh, bw, 8, 8), norm="ortho", axes=(-2, -1)) + 128.0
        out.append(np.clip(np.floor(v + 0.5), 0, 255).transpose(0, 2, 1, 3).reshape(bh * 8, bw * 8))
    return out


@pytest.mark.parametrize("mode", SAMPLINGS)
@pytest.mark.parametrize("ri", [0, 1, 3, 7])
def test_roundtrip_synth_encoder(mode, ri):
    qt = synth.quant_tables(75)
    rng = np.random.default_rng(11 + ri)
    for (w, h) in [(37, 29), (64, 48), (121, 83)]:
        im = synth.make_image(rng, w, h, qt, mode)
        b = jpeg.encode(im, qt, ri)
        info, planes, q2 = oracle.jpeg_decode(b)
        assert (info.width, info.height, info.ncomp, info.restart_interval) == (w, h, len(im.coef), ri)
        for c, p in enumerate(planes):
            assert np.array_equal(p, im.coef[c]), (mode, ri, w, h, c)
        assert np.array_equal(q2[0], qt[0])


def test_roundtrip_q95_dense_coefficients():
    qt = synth.quant_tables(95)
    im = synth.make_image(np.random.default_rng(5), 200, 120, qt, "natural")
    b = jpeg.encode(im, qt, 5)
    _, planes, _ = oracle.jpeg_decode(b)
    assert all(np.array_equal(p, c) for p, c in zip(planes, im.coef))


def _pil_jpeg(rgb, **kw):
    from PIL import Image
    buf = io.BytesIO()
    Image.fromarray(rgb).save(buf, "JPEG", **kw)
    return buf.getvalue()


@pytest.mark.parametrize("kw", [dict(quality=75, subsampling=2),
                                dict(quality=90, subsampling=0, restart_marker_blocks=5),
                                dict(quality=80, subsampling=1, restart_marker_rows=1),
                                dict(quality=75, subsampling=2, restart_marker_blocks=1)])
def test_libjpeg_files(kw):
    """Files from libjpeg's encoder: oracle coefficients -> plain IDCT ==
    libjpeg's own decoded samples within +-1 (its ISLOW integer IDCT)."""
    from PIL import Image
    rgb = synth.natural_rgb(np.random.default_rng(3), 150, 97)
    b = _pil_jpeg(rgb, **kw)
    info, planes, qt = oracle.jpeg_decode(b)
    assert (info.width, info.height) == (150, 97)
    if "restart_marker_blocks" in kw or "restart_marker_rows" in kw:
        assert info.restart_interval > 0
    ours = _idct_planes(planes, qt, list(info.tq))
    im = Image.open(io.BytesIO(b))
    im.draft("YCbCr", im.size)
    ycc = np.asarray(im.convert("YCbCr") if im.mode != "YCbCr" else im).astype(np.float64)
    assert np.abs(ours[0][:97, :150] - ycc[..., 0]).max() <= 1
    if kw.get("subsampling") == 0:            # 4:4:4: chroma planes are not resampled
        for c in (1, 2):
            assert np.abs(ours[c][:97, :150] - ycc[..., c]).max() <= 1


def test_libjpeg_gray_file():
    from PIL import Image
    rgb = synth.natural_rgb(np.random.default_rng(4), 77, 130)
    gray = np.asarray(Image.fromarray(rgb).convert("L"))
    buf = io.BytesIO()
    Image.fromarray(gray).save(buf, "JPEG", quality=85, restart_marker_blocks=3)
    b = buf.getvalue()
    info, planes, qt = oracle.jpeg_decode(b)
    assert info.ncomp == 1 and info.restart_interval == 3
    ours = _idct_planes(planes, qt, list(info.tq))[0][:130, :77]
    assert np.abs(ours - np.asarray(Image.open(io.BytesIO(b))).astype(np.float64)).max() <= 1


@pytest.mark.parametrize("mode", SAMPLINGS)
def test_libjpeg_decodes_synth_files(mode):
    """libjpeg reads synth's files to within +-1 of the plain IDCT of the
    planes synth encoded (the encoder writes a standard stream)."""
    from PIL import Image
    qt = synth.quant_tables(75)
    im = synth.make_image(np.random.default_rng(8), 90, 61, qt, mode)
    b = jpeg.encode(im, qt, 4)
    ref = _idct_planes(im.coef, qt, list(im.qidx))
    pim = Image.open(io.BytesIO(b))
    pim.draft("YCbCr" if not im.gray else "L", pim.size)
    got = np.asarray(pim).astype(np.float64)
    y = got if im.gray else got[..., 0]
    assert np.abs(ref[0][:61, :90] - y).max() <= 1


def test_zigzag_is_figure_a6():
    # the encoder's generated order: first entries of Figure A.6 and its
    # defining property (anti-diagonals alternate direction)
    zz = jpeg.ZIGZAG
    assert list(zz[:10]) == [0, 1, 8, 16, 9, 2, 3, 10, 17, 24] and zz[63] == 63
    assert sorted(zz) == list(range(64))
    s = [(i // 8) + (i % 8) for i in zz]
    assert s == sorted(s)


def test_rejects_bad_streams():
    qt = synth.quant_tables(75)
    im = synth.make_image(np.random.default_rng(1), 40, 40, qt, "natural")
    b = jpeg.encode(im, qt, 2)
    with pytest.raises(ValueError):
        oracle.jpeg_decode(b[:-200])                        # truncated scan
    with pytest.raises(ValueError):
        oracle.jpeg_decode(b"\x00\x01" + b[2:])             # no SOI
    prog = _pil_jpeg(synth.natural_rgb(np.random.default_rng(2), 32, 32), quality=75, progressive=True)
    with pytest.raises(ValueError):
        oracle.jpeg_decode(prog)                            # SOF2: not baseline
    bad = bytearray(b)                                      # wrong RST index
    k = bytes(bad).find(b"\xff\xd0")
    bad[k + 1] = 0xD3
    with pytest.raises(ValueError):
        oracle.jpeg_decode(bytes(bad))
