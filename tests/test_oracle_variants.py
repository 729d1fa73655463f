"""Pins of the oracle's decoder variants against things
other than the oracle itself:

* 4:2:2 / 4:4:4 chroma (reading R2 per axis, T.81 A.1.1 component sizes):
  4:4:4 is the identity (16 C in 1/16 units); modes agree where the
  mathematics says they must (vertically constant chroma: 4:2:0 == 4:2:2;
  horizontally constant: 4:2:2 == 4:4:4); brute-force per-pixel loops; the
  whole pipeline against an independent scipy / numpy / torch /
  torchvision reconstruction.
* Definition B reduced-scale IDCT (reading R16): scipy idctn(ortho) of
  (N/8) D[:N, :N]; DC-only closed form DC Q / 8 at every scale; equal to
  Definition A at 1/8; single-basis closed forms; the exact u = N/2 tie
  path.
* ROI rectangle (reading R15): the
  oracle's decoded RGB cropped to the window and resized with torchvision
  resized_crop (antialias off); a full-image window resized to the decoded
  size is the identity.
"""
import numpy as np
import pytest
import torch
import torch.nn.functional as F
from scipy import fft

import synth

MEAN = (0.485, 0.456, 0.406)
STD = (0.229, 0.224, 0.225)
HV = {420: (2, 2), 422: (2, 1), 444: (1, 1)}


# ----------------------------------------------------- independent pieces --
def _decode_planes_scipy(im, qt, k, idct_def="box"):
    """u8 planes by scipy: 8x8 orthonormal IDCT + k x k box mean (A), or the
    N-point orthonormal IDCT of (N/8) D[:N,:N] (B)."""
    hs, vs = HV[im.subsampling]
    W, H = im.width, im.height
    dims = [(-(-W // k), -(-H // k)), (-(-W // (hs * k)), -(-H // (vs * k)))]
    out = []
    for ci in range(3):
        c = im.coef[ci].astype(np.float64) * qt[im.qidx[ci]].astype(np.float64)
        bh, bw = c.shape[:2]
        c = c.reshape(bh, bw, 8, 8)
        P = 8 // k
        if idct_def == "box":
            s = fft.idctn(c, norm="ortho", axes=(-2, -1))
            s = s.reshape(bh, bw, P, k, P, k).mean(axis=(3, 5))
        else:
            s = fft.idctn(c[..., :P, :P] * (P / 8.0), norm="ortho", axes=(-2, -1))
        img = s.transpose(0, 2, 1, 3).reshape(bh * P, bw * P)
        w, h = dims[min(ci, 1)]
        x = img[:h, :w] + 128.5
        xr = np.rint(x)
        x = np.where(np.abs(x - xr) < 1e-9, xr, x)      # exact ties (R3) despite scipy noise
        out.append(np.clip(np.floor(x), 0, 255).astype(np.int64))
    return out


def _upsample_np(C, Wd, Hd, hs, vs):
    """Per-axis filter, vectorized: factor 2 -> 3/4, 1/4 (edge-clamped
    neighbour), factor 1 -> identity; result in 1/16 units."""
    def axis_idx(n_out, n_in, f):
        xs = np.arange(n_out)
        if f == 1:
            i = np.minimum(xs, n_in - 1)
            return i, i, 4, 0
        i = np.minimum(xs // 2, n_in - 1)
        i2 = np.clip(np.where(xs % 2 == 0, xs // 2 - 1, xs // 2 + 1), 0, n_in - 1)
        return i, i2, 3, 1
    Hc, Wc = C.shape
    i, i2, wx, wx2 = axis_idx(Wd, Wc, hs)
    j, j2, wy, wy2 = axis_idx(Hd, Hc, vs)
    h = wx * C[:, i] + wx2 * C[:, i2]
    return wy * h[j, :] + wy2 * h[j2, :]


def _colour_np(Y, cb16, cr16):
    den = 2_000_000
    db, dr = cb16 - 2048, cr16 - 2048
    R = np.floor_divide(den * Y + 175250 * dr + den // 2, den)
    G = np.floor_divide(den * Y - 43017 * db - 89267 * dr + den // 2, den)
    B = np.floor_divide(den * Y + 221500 * db + den // 2, den)
    return np.clip(np.stack([R, G, B]), 0, 255).astype(np.float64)


def independent_pipeline(im, qt, k, Wr, Hr, idct_def="box", roi_rect=None, chroma_2s=False):
    import torchvision.transforms.functional as TF
    hs, vs = HV[im.subsampling]
    Y, Cb, Cr = _decode_planes_scipy(im, qt, k, idct_def)
    Hd, Wd = Y.shape
    if chroma_2s:
        # reading R18: chroma decoded at 1/(k/2) onto the luma grid, no upsampling
        _, Cb, Cr = _decode_planes_scipy(im, qt, k // 2, idct_def)
        Cb, Cr = Cb[:Hd, :Wd], Cr[:Hd, :Wd]
        hs = vs = 1
    rgb = _colour_np(Y, _upsample_np(Cb, Wd, Hd, hs, vs), _upsample_np(Cr, Wd, Hd, hs, vs))
    t = torch.from_numpy(rgb)
    if roi_rect is not None:
        x, y, w, h = roi_rect
        x0, y0 = x // k, y // k
        x1, y1 = -(-(x + w) // k), -(-(y + h) // k)
        r = TF.resized_crop(t, y0, x0, y1 - y0, x1 - x0, [Hr, Wr],
                            interpolation=TF.InterpolationMode.BILINEAR, antialias=False)
    else:
        r = F.interpolate(t[None], size=(Hr, Wr), mode="bilinear", align_corners=False, antialias=False)[0]
    return TF.normalize(r / 255.0, MEAN, STD).numpy().astype(np.float32)


# ------------------------------------------------------------- subsampling --
@pytest.mark.parametrize("ss", [422, 444])
def test_encoder_shapes(ss):
    hs, vs = HV[ss]
    rng = np.random.default_rng(ss)
    qt = synth.quant_tables(75)
    for (w, h) in [(64, 48), (97, 61), (33, 17)]:
        im = synth.make_image(rng, w, h, qt, f"natural{ss}")
        assert im.subsampling == ss
        mh, mw = -(-h // (8 * vs)), -(-w // (8 * hs))
        assert im.coef[0].shape[:2] == (vs * mh, hs * mw)
        assert im.coef[1].shape[:2] == (mh, mw) == im.coef[2].shape[:2]


def test_444_upsample_is_identity(oracle_mod):
    rng = np.random.default_rng(1)
    for (w, h) in [(13, 7), (32, 32)]:
        Y = rng.integers(0, 256, (h, w), dtype=np.uint8)
        Cb = rng.integers(0, 256, (h, w), dtype=np.uint8)
        Cr = rng.integers(0, 256, (h, w), dtype=np.uint8)
        c16, _ = oracle_mod.upsample_color(Y, Cb, Cr, 444)
        np.testing.assert_array_equal(c16[..., 0], 16 * Cb.astype(np.int32))
        np.testing.assert_array_equal(c16[..., 1], 16 * Cr.astype(np.int32))


def test_modes_agree_where_they_must(oracle_mod):
    """Vertically constant chroma: 4:2:0 and 4:2:2 both reduce to the
    horizontal triangle; horizontally constant chroma: 4:2:2 (vertical
    identity, horizontal filter of a constant) equals 4:4:4."""
    rng = np.random.default_rng(2)
    Wd, Hd = 22, 14
    Y = rng.integers(0, 256, (Hd, Wd), dtype=np.uint8)
    row = rng.integers(0, 256, (1, 11), dtype=np.uint8)
    c420 = np.repeat(row, 7, axis=0)            # Hc = 7 for 4:2:0
    c422 = np.repeat(row, 14, axis=0)           # Hc = 14 for 4:2:2
    a, ra = oracle_mod.upsample_color(Y, c420, c420[::-1].copy(), 420)
    b, rb = oracle_mod.upsample_color(Y, c422, c422[::-1].copy(), 422)
    np.testing.assert_array_equal(a, b)
    np.testing.assert_array_equal(ra, rb)
    col = rng.integers(0, 256, (Hd, 1), dtype=np.uint8)
    d422 = np.repeat(col, 11, axis=1)
    d444 = np.repeat(col, 22, axis=1)
    c, rc = oracle_mod.upsample_color(Y, d422, d422, 422)
    d, rd = oracle_mod.upsample_color(Y, d444, d444, 444)
    np.testing.assert_array_equal(c, d)
    np.testing.assert_array_equal(rc, rd)


@pytest.mark.parametrize("ss", [420, 422, 444])
def test_upsample_brute_force(oracle_mod, ss):
    """Per-pixel loops over the per-axis rule (clamped neighbours)."""
    hs, vs = HV[ss]
    rng = np.random.default_rng(3 + ss)
    Wd, Hd = 9, 7
    Wc, Hc = -(-Wd // hs), -(-Hd // vs)
    C = rng.integers(0, 256, (Hc, Wc)).astype(np.int64)
    Y = np.zeros((Hd, Wd), np.uint8)
    c16, _ = oracle_mod.upsample_color(Y, C.astype(np.uint8), C.astype(np.uint8), ss)
    for y in range(Hd):
        for x in range(Wd):
            def taps(p, f, n):
                if f == 1:
                    return [(min(p, n - 1), 4)]
                i = min(p // 2, n - 1)
                i2 = p // 2 - 1 if p % 2 == 0 else p // 2 + 1
                return [(i, 3), (min(max(i2, 0), n - 1), 1)]
            want = sum(wy * wx * C[j, i] for j, wy in taps(y, vs, Hc) for i, wx in taps(x, hs, Wc))
            assert c16[y, x, 0] == want, (ss, y, x)


@pytest.mark.parametrize("ss", [422, 444])
@pytest.mark.parametrize("k", [1, 2, 4, 8])
def test_pipeline_subsampling_vs_independent(oracle_mod, ss, k):
    rng = np.random.default_rng(500 + ss + k)
    qt = synth.quant_tables(75)
    for (w, h) in [(64, 48), (41, 23), (16, 16)]:
        im = synth.make_image(rng, w, h, qt, f"natural{ss}")
        p = oracle_mod.make_params(scale_denom=k, resize_mode="exact", resize_w=13, resize_h=11)
        got = oracle_mod.run_image(p, im, qt)
        ref = independent_pipeline(im, qt, k, 13, 11)
        assert np.max(np.abs(got - ref)) < 2e-6, (ss, k, w, h)


def test_subsampling_geometry(oracle_mod):
    p = oracle_mod.make_params(scale_denom=2, resize_mode="exact", resize_w=8, resize_h=8)
    for ss, (wc, hc) in [(420, (125, 94)), (422, (125, 188)), (444, (250, 188))]:
        g = oracle_mod.geometry(p, 500, 375, ss)
        assert (g.Wd, g.Hd, g.Wc, g.Hc) == (250, 188, wc, hc)


# ------------------------------------------------------------ Definition B --
@pytest.mark.parametrize("k", [2, 4, 8])
def test_def_b_vs_scipy(oracle_mod, k):
    rng = np.random.default_rng(600 + k)
    P = 8 // k
    for _ in range(20):
        c = rng.integers(-60, 61, (2, 3, 64)).astype(np.int16)
        q = rng.integers(1, 40, 64).astype(np.uint16)
        v, _ = oracle_mod.decode_plane(c, q, k, 3 * P, 2 * P, idct_def=1)
        D = (c.astype(np.float64) * q).reshape(2, 3, 8, 8)
        ref = fft.idctn(D[..., :P, :P] * (P / 8.0), norm="ortho", axes=(-2, -1))
        ref = ref.transpose(0, 2, 1, 3).reshape(2 * P, 3 * P)
        assert np.max(np.abs(v - ref)) < 1e-11


@pytest.mark.parametrize("k", [2, 4, 8])
def test_def_b_dc_closed_form(oracle_mod, k):
    """DC-only block: every sample = floor(DC Q / 8 + 128.5), as Definition A."""
    P = 8 // k
    q = np.ones(64, np.uint16)
    dcs = np.arange(-2048, 2048, dtype=np.int64)
    c = np.zeros((1, dcs.size, 64), np.int16)
    c[0, :, 0] = dcs
    _, u8 = oracle_mod.decode_plane(c, q, k, dcs.size * P, P, idct_def=1)
    want = np.clip(np.floor(dcs / 8.0 + 128.5), 0, 255)
    for j in range(P):
        np.testing.assert_array_equal(u8[:, j::P].astype(np.int64), np.tile(want, (P, 1)))


def test_def_b_equals_a_at_one_eighth(oracle_mod):
    rng = np.random.default_rng(8)
    c = rng.integers(-300, 300, (5, 7, 64)).astype(np.int16)
    q = rng.integers(1, 60, 64).astype(np.uint16)
    va, ua = oracle_mod.decode_plane(c, q, 8, 7, 5, idct_def=0)
    vb, ub = oracle_mod.decode_plane(c, q, 8, 7, 5, idct_def=1)
    np.testing.assert_array_equal(ua, ub)
    np.testing.assert_array_equal(va, vb)


@pytest.mark.parametrize("k", [2, 4])
def test_def_b_single_basis_and_exact_tie(oracle_mod, k):
    """One coefficient D(v,u) (u, v < N) gives 1/8 D b_N(v,i) b_N(u,j),
    b_N(u,x) = sqrt2 C(u) cos((2x+1) u pi / 2N); the u = N/2 entries are
    exactly +-1, so D(0, N/2) = 4 gives the exact ties 128 +- 1/2 ->
    129 / 128 (round half up)."""
    N = 8 // k
    q = np.ones(64, np.uint16)

    def b(u, x):
        return 1.0 if u == 0 else np.sqrt(2.0) * np.cos((2 * x + 1) * u * np.pi / (2 * N))
    for vv in range(N):
        for uu in range(N):
            c = np.zeros((1, 1, 64), np.int16)
            c[0, 0, vv * 8 + uu] = 40
            v, _ = oracle_mod.decode_plane(c, q, k, N, N, idct_def=1)
            ref = np.array([[40 / 8 * b(vv, i) * b(uu, j) for j in range(N)] for i in range(N)])
            assert np.max(np.abs(v - ref)) < 1e-12
    c = np.zeros((1, 1, 64), np.int16)
    c[0, 0, N // 2] = 4
    v, u8 = oracle_mod.decode_plane(c, q, k, N, N, idct_def=1)
    sign = np.array([1.0 if ((2 * x + 1) % 8) in (1, 7) else -1.0 for x in range(N)])
    np.testing.assert_array_equal(v, np.tile(0.5 * sign, (N, 1)))
    np.testing.assert_array_equal(u8, np.tile(np.where(sign > 0, 129, 128), (N, 1)))


@pytest.mark.parametrize("k", [2, 4])
def test_def_b_pipeline_vs_independent(oracle_mod, k):
    rng = np.random.default_rng(700 + k)
    qt = synth.quant_tables(75)
    for (w, h, ss) in [(64, 48, 420), (41, 23, 444), (48, 40, 422)]:
        im = synth.make_image(rng, w, h, qt, "natural" if ss == 420 else f"natural{ss}")
        p = oracle_mod.make_params(scale_denom=k, resize_mode="exact", resize_w=13, resize_h=11,
                                   idct_def="truncated")
        got = oracle_mod.run_image(p, im, qt)
        ref = independent_pipeline(im, qt, k, 13, 11, idct_def="truncated")
        assert np.max(np.abs(got - ref)) < 2e-6, (k, w, h, ss)


# ------------------------------------------------------------ ROI rectangle --
@pytest.mark.parametrize("k", [1, 2, 4])
def test_roi_rect_vs_torchvision_resized_crop(oracle_mod, k):
    rng = np.random.default_rng(800 + k)
    qt = synth.quant_tables(75)
    for (w, h, rect) in [(64, 48, (10, 7, 30, 20)), (97, 61, (0, 0, 97, 61)), (80, 80, (33, 41, 17, 9)),
                         (64, 48, (5, 3, 58, 44))]:
        im = synth.make_image(rng, w, h, qt)
        p = oracle_mod.make_params(scale_denom=k, resize_mode="exact", resize_w=24, resize_h=16)
        got = oracle_mod.run_image(p, im, qt, roi_rect=rect)
        ref = independent_pipeline(im, qt, k, 24, 16, roi_rect=rect)
        assert got.shape == (3, 16, 24)
        assert np.max(np.abs(got - ref)) < 2e-6, (k, w, h, rect)


def test_roi_rect_full_window_identity(oracle_mod):
    """Whole image as the window, resized to its own decoded size: the
    output is the normalized decoded RGB (bilinear identity, R8)."""
    rng = np.random.default_rng(9)
    qt = synth.quant_tables(75)
    im = synth.make_image(rng, 40, 24, qt)
    p = oracle_mod.make_params(scale_denom=2, resize_mode="exact", resize_w=20, resize_h=12)
    got = oracle_mod.run_image(p, im, qt, roi_rect=(0, 0, 40, 24))
    Y, Cb, Cr = oracle_mod.decode_image_planes(p, im, qt)
    _, rgb = oracle_mod.upsample_color(Y, Cb, Cr)
    want = (rgb.transpose(2, 0, 1) / 255.0 - np.array(MEAN)[:, None, None]) / np.array(STD)[:, None, None]
    np.testing.assert_allclose(got, want.astype(np.float32), rtol=0, atol=1e-6)


def test_roi_rect_window_rounding(oracle_mod):
    """Reading R15: the SOF rectangle maps to [floor(x/k), ceil((x+w)/k)) --
    a rectangle and its decoded-aligned cover give the same output."""
    rng = np.random.default_rng(10)
    qt = synth.quant_tables(75)
    im = synth.make_image(rng, 64, 64, qt)
    p = oracle_mod.make_params(scale_denom=4, resize_mode="exact", resize_w=8, resize_h=8)
    a = oracle_mod.run_image(p, im, qt, roi_rect=(5, 9, 22, 13))      # -> [1, 7) x [2, 6)
    b = oracle_mod.run_image(p, im, qt, roi_rect=(4, 8, 24, 16))      # exactly [1, 7) x [2, 6)
    np.testing.assert_array_equal(a, b)


# ------------------------------------------------- chroma at twice the scale --
@pytest.mark.parametrize("k", [2, 4, 8])
def test_chroma_2s_vs_independent(oracle_mod, k):
    """Reading R18 (libjpeg-turbo scaled decoding of 4:2:0): chroma blocks
    decoded at 1/(k/2) land on the luma grid and are used without
    upsampling -- against scipy box means at k/2 and the identity filter."""
    rng = np.random.default_rng(1000 + k)
    qt = synth.quant_tables(75)
    for (w, h) in [(64, 48), (97, 61), (40, 40)]:
        im = synth.make_image(rng, w, h, qt)
        p = oracle_mod.make_params(scale_denom=k, resize_mode="exact", resize_w=13, resize_h=11, chroma_2s=True)
        got = oracle_mod.run_image(p, im, qt)
        ref = independent_pipeline(im, qt, k, 13, 11, chroma_2s=True)
        assert np.max(np.abs(got - ref)) < 2e-6, (k, w, h)
        Y, Cb, Cr = oracle_mod.decode_image_planes(p, im, qt)
        assert Cb.shape == Y.shape == (-(-h // k), -(-w // k))


def test_chroma_2s_equals_r2_on_constant_chroma(oracle_mod):
    """With one chroma level everywhere both readings give the same image
    (triangle of a constant = the constant; DC-only blocks decode to DC/8 at
    any scale)."""
    qt = synth.quant_tables(75)
    rng = np.random.default_rng(7)
    im = synth.make_image(rng, 64, 48, qt)
    coef = [im.coef[0]] + [np.zeros_like(c) for c in im.coef[1:]]
    coef[1][..., 0] = 5
    coef[2][..., 0] = -3
    im2 = synth.CoefImage(64, 48, coef)
    for k in (2, 4, 8):
        a = oracle_mod.run_image(oracle_mod.make_params(scale_denom=k, resize_mode="exact", resize_w=16, resize_h=12), im2, qt)
        b = oracle_mod.run_image(oracle_mod.make_params(scale_denom=k, resize_mode="exact", resize_w=16, resize_h=12,
                                                        chroma_2s=True), im2, qt)
        np.testing.assert_array_equal(a, b)
