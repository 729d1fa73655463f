"""Pins for the oracle's 4:2:0 upsample and JFIF colour conversion.

Colour is pinned against exact rational arithmetic (fractions.Fraction) on the
complete list of exact ties plus random samples; upsampling against constant,
linear-ramp and mirror-symmetry properties (reading R2).
"""
import json
import os
from fractions import Fraction as Fr

import numpy as np

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def jfif_fraction(Y, cb16, cr16):
    """JFIF 1.02 with decimal constants, exactly; round half up; clamp."""
    cb = Fr(cb16, 16) - 128
    cr = Fr(cr16, 16) - 128
    R = Y + Fr("1.402") * cr
    G = Y - Fr("0.344136") * cb - Fr("0.714136") * cr
    B = Y + Fr("1.772") * cb
    f = lambda x: max(0, min(255, int((x + Fr(1, 2)).__floor__())))
    return f(R), f(G), f(B)


def test_color_worked_pins(oracle_mod):
    pins = json.load(open(os.path.join(GOLD, "survey_pins.json")))["color"]
    for p in pins:
        Y, cb, cr = p["ycc"]
        assert jfif_fraction(Y, 16 * cb, 16 * cr) == tuple(p["rgb"])
        assert oracle_mod.color(Y, 16 * cb, 16 * cr) == tuple(p["rgb"])


def test_color_gray_axis(oracle_mod):
    for Y in range(256):
        assert oracle_mod.color(Y, 2048, 2048) == (Y, Y, Y)


def test_color_all_exact_ties(oracle_mod):
    # Exact ties: integer chroma B at Cb-128 = +-125, G at
    # (Cb-128, Cr-128) = (-+50, +-50); in 1/16 units (+-800, -+800),
    # (+-791, +-459), (+-782, +-1718).  Enumerate every (d16b, d16r) whose R, G
    # or B fraction part is exactly 1/2 for some Y, by brute force, and check.
    ties = set()
    for db in range(-2048, 2033):
        # B = Y + 0.11075 d16b: half-integer iff 110750*db = 500000 mod 10^6 ... check via Fraction
        if (Fr("1.772") * Fr(db, 16)).denominator == 2:
            for dr in (-2048, 0, 2032):
                ties.add((db, dr))
    for dr in range(-2048, 2033):
        if (Fr("1.402") * Fr(dr, 16)).denominator == 2:
            ties.add((0, dr))
    cands = [(800, -800), (-800, 800), (791, 459), (-791, -459), (782, 1718), (-782, -1718)]
    for db, dr in cands:
        g = -Fr("0.344136") * Fr(db, 16) - Fr("0.714136") * Fr(dr, 16)
        assert g.denominator == 2, (db, dr)
        ties.add((db, dr))
    assert len(ties) > 6
    for db, dr in sorted(ties):
        if not (0 <= db + 2048 <= 4080 and 0 <= dr + 2048 <= 4080):
            continue
        for Y in range(0, 256, 5):
            assert oracle_mod.color(Y, db + 2048, dr + 2048) == jfif_fraction(Y, db + 2048, dr + 2048)


def test_color_random_vs_fraction(oracle_mod):
    rng = np.random.default_rng(7)
    for _ in range(20000):
        Y = int(rng.integers(0, 256))
        cb, cr = (int(x) for x in rng.integers(0, 4081, size=2))
        assert oracle_mod.color(Y, cb, cr) == jfif_fraction(Y, cb, cr)


def _up(oracle_mod, Cb, Cr, Wd, Hd, Y=None):
    Y = np.full((Hd, Wd), 128, np.uint8) if Y is None else Y
    return oracle_mod.upsample_color(Y, Cb, Cr)


def test_upsample_constant(oracle_mod):
    for (Wd, Hd) in [(16, 16), (15, 9), (1, 1), (2, 3)]:
        Wc, Hc = (Wd + 1) // 2, (Hd + 1) // 2
        Cb = np.full((Hc, Wc), 77, np.uint8)
        Cr = np.full((Hc, Wc), 201, np.uint8)
        c16, _ = _up(oracle_mod, Cb, Cr, Wd, Hd)
        assert np.all(c16[..., 0] == 16 * 77) and np.all(c16[..., 1] == 16 * 201)


def test_upsample_linear_ramp_centered_siting(oracle_mod):
    # Chroma sample i sits at luma x = 2i + 1/2; a linear ramp C[i] = a + b i is
    # reproduced in the interior: c16(X) = 16 (a + b (X - 1/2) / 2).
    Wd, Hd = 32, 20
    Wc, Hc = 16, 10
    i = np.arange(Wc)
    Cb = np.tile((10 + 8 * i).astype(np.uint8), (Hc, 1))            # horizontal ramp
    Cr = np.tile((20 + 12 * np.arange(Hc)).astype(np.uint8)[:, None], (1, Wc))  # vertical
    c16, _ = _up(oracle_mod, Cb, Cr, Wd, Hd)
    X = np.arange(Wd)
    exp_b = 16 * (10 + 8 * (X - 0.5) / 2)
    for y in range(Hd):
        assert np.array_equal(c16[y, 1:Wd - 1, 0], exp_b[1:Wd - 1])
    Yr = np.arange(Hd)
    exp_r = 16 * (20 + 12 * (Yr - 0.5) / 2)
    for x in range(Wd):
        assert np.array_equal(c16[1:Hd - 1, x, 1], exp_r[1:Hd - 1])
    # edges replicate the border chroma sample (index clamped)
    assert np.all(c16[:, 0, 0] == 16 * 10) and np.all(c16[:, Wd - 1, 0] == 16 * (10 + 8 * (Wc - 1)))


def test_upsample_mirror_symmetry(oracle_mod):
    rng = np.random.default_rng(11)
    Wd, Hd = 24, 14
    Cb = rng.integers(0, 256, size=(7, 12)).astype(np.uint8)
    Cr = rng.integers(0, 256, size=(7, 12)).astype(np.uint8)
    c16, _ = _up(oracle_mod, Cb, Cr, Wd, Hd)
    c16m, _ = _up(oracle_mod, Cb[:, ::-1].copy(), Cr[::-1, :].copy(), Wd, Hd)
    assert np.array_equal(c16m[:, :, 0], c16[:, ::-1, 0])
    assert np.array_equal(c16m[:, :, 1], c16[::-1, :, 1])


def test_upsample_weights_sum_and_brute(oracle_mod):
    # Brute force on a tiny plane: explicit 9/3/3/1 neighbours with clamping.
    rng = np.random.default_rng(12)
    Wd, Hd = 7, 5
    Wc, Hc = 4, 3
    Cb = rng.integers(0, 256, size=(Hc, Wc)).astype(np.uint8)
    c16, _ = _up(oracle_mod, Cb, Cb, Wd, Hd)
    cl = lambda a, n: min(max(a, 0), n - 1)
    for Y in range(Hd):
        for X in range(Wd):
            i, j = X // 2, Y // 2
            i2 = cl(i - 1 if X % 2 == 0 else i + 1, Wc)
            j2 = cl(j - 1 if Y % 2 == 0 else j + 1, Hc)
            e = 9 * int(Cb[j, i]) + 3 * int(Cb[j, i2]) + 3 * int(Cb[j2, i]) + int(Cb[j2, i2])
            assert c16[Y, X, 0] == e


def test_upsample_color_composes(oracle_mod):
    rng = np.random.default_rng(13)
    Y = rng.integers(0, 256, size=(6, 8)).astype(np.uint8)
    Cb = rng.integers(0, 256, size=(3, 4)).astype(np.uint8)
    Cr = rng.integers(0, 256, size=(3, 4)).astype(np.uint8)
    c16, rgb = oracle_mod.upsample_color(Y, Cb, Cr)
    for y in range(6):
        for x in range(8):
            assert tuple(rgb[y, x]) == jfif_fraction(int(Y[y, x]), int(c16[y, x, 0]), int(c16[y, x, 1]))
