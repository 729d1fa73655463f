"""Pins for the oracle's resize / crop / normalize and geometry.

Bilinear is pinned against torch.nn.functional.interpolate in float64
(align_corners=False, antialias=False -- reading R8); resize/crop geometry
against torchvision's own functional resize / center_crop (reading R7);
normalization against closed forms; Algorithm 1 against the SPEC
worked example (tests/golden/alg1_window.json).
"""
import json
import os

import numpy as np
import pytest
import torch
import torch.nn.functional as F

GOLD = os.path.join(os.path.dirname(__file__), "golden")
MEAN = (0.485, 0.456, 0.406)
STD = (0.229, 0.224, 0.225)
ID_MEAN, ID_STD = (0.0, 0.0, 0.0), (1 / 255, 1 / 255, 1 / 255)


def _resize(oracle_mod, rgb, Wr, Hr):
    _, res = oracle_mod.resize_crop_normalize(rgb, Wr, Hr, 0, 0, Wr, Hr, ID_MEAN, ID_STD)
    return res


@pytest.mark.parametrize("src,dst", [((375, 500), (256, 341)), ((188, 250), (256, 340)),
                                     ((94, 125), (256, 340)), ((21, 21), (64, 64)),
                                     ((270, 480), (224, 224)), ((64, 64), (32, 32)),
                                     ((37, 53), (37, 53)), ((61, 97), (200, 13))])
def test_bilinear_matches_torch_f64(oracle_mod, src, dst):
    rng = np.random.default_rng(hash(src + dst) % 2 ** 32)
    Hd, Wd = src
    Hr, Wr = dst
    rgb = rng.integers(0, 256, size=(Hd, Wd, 3)).astype(np.uint8)
    res = _resize(oracle_mod, rgb, Wr, Hr)
    t = torch.from_numpy(rgb.astype(np.float64)).permute(2, 0, 1)[None]
    ref = F.interpolate(t, size=(Hr, Wr), mode="bilinear", align_corners=False, antialias=False)[0].numpy()
    assert np.max(np.abs(res - ref)) < 1e-9


def test_identity_and_half(oracle_mod):
    rng = np.random.default_rng(21)
    rgb = rng.integers(0, 256, size=(20, 30, 3)).astype(np.uint8)
    assert np.array_equal(_resize(oracle_mod, rgb, 30, 20), rgb.transpose(2, 0, 1).astype(np.float64))
    half = _resize(oracle_mod, rgb, 15, 10)
    mean2 = rgb.astype(np.float64).reshape(10, 2, 15, 2, 3).mean(axis=(1, 3)).transpose(2, 0, 1)
    assert np.max(np.abs(half - mean2)) < 1e-12


def test_normalize_closed_forms(oracle_mod):
    pins = json.load(open(os.path.join(GOLD, "survey_pins.json")))
    for c in (0, 1, 77, 128, 255):
        rgb = np.full((4, 4, 3), c, np.uint8)
        out, _ = oracle_mod.resize_crop_normalize(rgb, 4, 4, 0, 0, 4, 4, MEAN, STD)
        for ch in range(3):
            exp = np.float32((c / 255 - MEAN[ch]) / STD[ch])
            assert np.all(out[ch] == exp)
    w, _ = oracle_mod.resize_crop_normalize(np.full((2, 2, 3), 255, np.uint8), 2, 2, 0, 0, 2, 2, MEAN, STD)
    b, _ = oracle_mod.resize_crop_normalize(np.zeros((2, 2, 3), np.uint8), 2, 2, 0, 0, 2, 2, MEAN, STD)
    assert np.allclose(w[:, 0, 0], pins["normalize_white"], atol=1e-6)
    assert np.allclose(b[:, 0, 0], pins["normalize_black"], atol=1e-6)


def test_f16_output_rne(oracle_mod):
    rng = np.random.default_rng(22)
    xs = np.concatenate([rng.uniform(-3, 3, 20000), rng.uniform(-1e-4, 1e-4, 2000),
                         [0.0, -0.0, 2.640, -2.1179039, 65504.0, 1e-8, 6.1e-5]])
    for x in xs:
        assert oracle_mod.f64_to_f16_bits(x) == int(np.float16(x).view(np.uint16)), x
    # halfway cases in [1, 2): ulp 2^-10, halfway -> even mantissa
    for m in range(0, 1024, 37):
        x = 1.0 + (m + 0.5) / 1024
        assert oracle_mod.f64_to_f16_bits(x) == int(np.float16(x).view(np.uint16))


def test_crop_window_offsets(oracle_mod):
    rng = np.random.default_rng(23)
    rgb = rng.integers(0, 256, size=(30, 40, 3)).astype(np.uint8)
    full = _resize(oracle_mod, rgb, 40, 30)
    _, crop = oracle_mod.resize_crop_normalize(rgb, 40, 30, 5, 3, 20, 11, ID_MEAN, ID_STD)
    assert np.array_equal(crop, full[:, 3:14, 5:25])


def test_decoded_dims(oracle_mod):
    pins = json.load(open(os.path.join(GOLD, "survey_pins.json")))
    for d in pins["decoded_dims"]:
        p = oracle_mod.make_params(scale_denom=d["k"], resize_mode="exact", resize_w=8, resize_h=8)
        g = oracle_mod.geometry(p, d["w"], d["h"])
        assert (g.Wd, g.Hd) == (d["Wd"], d["Hd"])
        assert (g.Wc, g.Hc) == (-(-d["w"] // (2 * d["k"])), -(-d["h"] // (2 * d["k"])))


def test_geometry_matches_torchvision(oracle_mod):
    import torchvision.transforms.functional as TF
    pins = json.load(open(os.path.join(GOLD, "survey_pins.json")))["c2_geometry"]
    rng = np.random.default_rng(24)
    sizes = [(500, 375), (375, 500), (333, 500), (161, 161), (1920, 1080), (256, 300), (257, 999)]
    sizes += [(int(a), int(b)) for a, b in rng.integers(230, 1200, size=(40, 2))]
    for (w, h) in sizes:
        p = oracle_mod.make_params(scale_denom=1, resize_short=256, crop_w=224, crop_h=224)
        g = oracle_mod.geometry(p, w, h)
        img = torch.zeros(1, h, w)
        r = TF.resize(img, 256, antialias=False)
        assert (g.Hr, g.Wr) == tuple(r.shape[-2:]), (w, h)
        # crop offsets: mark coordinates and read them back after center_crop
        yy, xx = torch.meshgrid(torch.arange(g.Hr), torch.arange(g.Wr), indexing="ij")
        marks = torch.stack([yy, xx]).float()
        cc = TF.center_crop(marks, [224, 224])
        assert (g.top, g.left) == (int(cc[0, 0, 0]), int(cc[1, 0, 0])), (w, h)
    p = oracle_mod.make_params(scale_denom=1, resize_short=256, crop_w=224, crop_h=224)
    g = oracle_mod.geometry(p, pins["w"], pins["h"])
    assert (g.Wr, g.Hr, g.left, g.top) == (pins["Wr"], pins["Hr"], pins["left"], pins["top"])


def test_algorithm1_window(oracle_mod):
    for c in json.load(open(os.path.join(GOLD, "alg1_window.json")))["cases"]:
        assert oracle_mod.alg1_crop_window(c["height"], c["width"], c["target"]) == (
            c["l"], c["r"], c["t"], c["b"])
