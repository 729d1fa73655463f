"""Pins for the oracle's dequantize + IDCT (+ reduced-scale) step.

Pinned against things other than the oracle itself: scipy's orthonormal
DCT-III (== T.81 A.3.3 IDCT), Parseval, libjpeg-turbo jidctred constants
(tests/golden/jidctred_constants.json), closed forms for DC-only blocks and
the SURVEY §8(c) worked pins (re-derived below).
"""
import json
import os

import numpy as np
import pytest
from scipy import fft

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _plane_of_blocks(blocks):
    """list of [64] -> coef plane [1][n][64] int16."""
    a = np.asarray(blocks, dtype=np.int16).reshape(1, -1, 64)
    return a


def _v_blocks(oracle_mod, coef, q, k):
    """Decode a [1][n][64] plane at 1/k; return v as [n][P][P]."""
    P = 8 // k
    n = coef.shape[1]
    v, u8 = oracle_mod.decode_plane(coef, q, k, n * P, P)
    return v.reshape(P, n, P).transpose(1, 0, 2), u8.reshape(P, n, P).transpose(1, 0, 2)


def test_idct_matches_scipy_orthonormal(oracle_mod):
    # T.81 A.3.3 IDCT == orthonormal 2-D DCT-III (scipy idctn norm='ortho').
    rng = np.random.default_rng(1)
    q = rng.integers(1, 40, size=64).astype(np.uint16)
    coef = rng.integers(-60, 61, size=(3, 5, 64)).astype(np.int16)   # 3x5 block grid
    v, _ = oracle_mod.decode_plane(coef, q, 1, 40, 24)
    for by in range(3):
        for bx in range(5):
            D = coef[by, bx].astype(np.float64) * q
            ref = fft.idctn(D.reshape(8, 8), norm="ortho")          # [y][x], D[v][u]
            got = v[by * 8:(by + 1) * 8, bx * 8:(bx + 1) * 8]
            assert np.max(np.abs(got - ref)) < 1e-9


def test_idct_block_layout_row_major_and_transpose(oracle_mod):
    # A horizontal-frequency coefficient (v=0, u=1) varies along x only.
    q = np.ones(64, np.uint16)
    c = np.zeros(64, np.int16)
    c[1] = 100                                     # natural order index v*8+u
    v, _ = _v_blocks(oracle_mod, _plane_of_blocks([c]), q, 1)
    assert np.allclose(v[0], v[0][0:1, :])         # rows identical
    assert not np.allclose(v[0][:, 0], v[0][:, 7])


def test_parseval(oracle_mod):
    rng = np.random.default_rng(2)
    q = np.ones(64, np.uint16)
    blocks = rng.integers(-300, 301, size=(16, 64))
    v, _ = _v_blocks(oracle_mod, _plane_of_blocks(blocks), q, 1)
    for b in range(16):
        assert abs((v[b] ** 2).sum() - (blocks[b].astype(np.float64) ** 2).sum()) < 1e-6 * (
            1 + (blocks[b].astype(np.float64) ** 2).sum())


def test_single_basis_closed_form(oracle_mod):
    # T.81 A.3.3 with one non-zero S(v,u)=c: s(y,x) = c/4 C(u)C(v) cos((2x+1)u pi/16) cos((2y+1)v pi/16)
    q = np.ones(64, np.uint16)
    C = lambda u: 1 / np.sqrt(2) if u == 0 else 1.0
    x = np.arange(8)
    for (vv, u) in [(0, 0), (0, 3), (5, 0), (2, 6), (7, 7), (4, 4), (1, 4)]:
        c = np.zeros(64, np.int16)
        c[vv * 8 + u] = 37
        got, _ = _v_blocks(oracle_mod, _plane_of_blocks([c]), q, 1)
        ref = 37 / 4 * C(u) * C(vv) * np.outer(np.cos((2 * x + 1) * vv * np.pi / 16),
                                              np.cos((2 * x + 1) * u * np.pi / 16))
        assert np.max(np.abs(got[0] - ref)) < 1e-12


@pytest.mark.parametrize("k", [1, 2, 4, 8])
def test_dc_only_closed_form_all_dc(oracle_mod, k):
    # DC-only block, Q=1: every sample = DC/8 (exact), u8 = clamp(floor(DC/8 + 128.5)).
    # north_star: "a DC-only block gives a constant DC/8+128"; "the 1/8-scale decode
    # equals DC/8+128".  All 4096 DC values of the 12-bit range.
    P = 8 // k
    dcs = np.arange(-2048, 2048)
    coef = np.zeros((64, 64, 64), np.int16)                  # 64x64 grid = 4096 blocks
    coef.reshape(-1, 64)[:, 0] = dcs
    q = np.ones(64, np.uint16)
    v, u8 = oracle_mod.decode_plane(coef, q, k, 64 * P, 64 * P)
    exp_v = (dcs / 8.0).reshape(64, 64)
    exp_u8 = np.clip(np.floor(dcs / 8.0 + 128.5), 0, 255).astype(np.uint8).reshape(64, 64)
    vb = v.reshape(64, P, 64, P)
    ub = u8.reshape(64, P, 64, P)
    assert np.array_equal(vb, np.broadcast_to(exp_v[:, None, :, None], vb.shape))   # exact
    assert np.array_equal(ub, np.broadcast_to(exp_u8[:, None, :, None], ub.shape))


def test_survey_worked_pins(oracle_mod):
    pins = json.load(open(os.path.join(GOLD, "survey_pins.json")))
    q = np.ones(64, np.uint16)
    for p in pins["dc_ties"] + pins["clamp"]:
        c = np.zeros(64, np.int16)
        c[0] = p["dc"]
        # closed form: v = dc/8; u8 = clamp(floor(v + 128 + 1/2))
        cf = int(np.clip(np.floor(p["dc"] / 8 + 128.5), 0, 255))
        assert cf == p["u8"]
        for k in (1, 8):
            _, u8 = _v_blocks(oracle_mod, _plane_of_blocks([c]), q, k)
            assert np.all(u8 == p["u8"])
    # u = 4 exact tie path: S(0,4) = 4 -> s(y,x) = 4/8 * t(4,x) = +-1/2 exactly,
    # t(4,x) = sqrt2 cos((2x+1)pi/4) = + for x in {0,3,4,7}, - otherwise.
    u4 = pins["u4_row"]
    c = np.zeros(64, np.int16)
    c[u4["coef_index"]] = u4["value"]
    v, u8 = _v_blocks(oracle_mod, _plane_of_blocks([c]), q, 1)
    assert set(np.abs(v[0]).ravel().tolist()) == {0.5}
    for y in range(8):
        assert u8[0][y].tolist() == u4["row"]
    # box mean over pairs cancels exactly: v = 0 -> 128 at scale 1/2
    v2, u82 = _v_blocks(oracle_mod, _plane_of_blocks([c]), q, 2)
    assert np.all(v2 == 0.0) and np.all(u82 == u4["half_scale"])


@pytest.mark.parametrize("k", [2, 4, 8])
def test_reduced_scale_is_box_mean_of_scipy_idct(oracle_mod, k):
    # Reading R1 (Definition A) against an independent IDCT (scipy).
    rng = np.random.default_rng(3 + k)
    q = rng.integers(1, 30, size=64).astype(np.uint16)
    blocks = rng.integers(-50, 51, size=(12, 64))
    v, _ = _v_blocks(oracle_mod, _plane_of_blocks(blocks), q, k)
    P = 8 // k
    for b in range(12):
        full = fft.idctn((blocks[b] * q.astype(np.float64)).reshape(8, 8), norm="ortho")
        ref = full.reshape(P, k, P, k).mean(axis=(1, 3))
        assert np.max(np.abs(v[b] - ref)) < 1e-9


def test_reduced_scale_matches_libjpeg_turbo_jidctred(oracle_mod):
    g = json.load(open(os.path.join(GOLD, "jidctred_constants.json")))
    tol = g["tolerance"]
    q = np.ones(64, np.uint16)
    c0 = 1000
    for k, J, div in ((2, g["J4x4"], 16.0), (4, g["J2x2"], 32.0)):
        P = 8 // k
        for u in range(8):
            c = np.zeros(64, np.int16)
            c[u] = c0                                 # S(v=0, u)
            v, _ = _v_blocks(oracle_mod, _plane_of_blocks([c]), q, k)
            for j in range(P):
                # rows of J cover output columns j < len(J); the rest mirror with
                # odd-u sign flips (J[P-1-j][u] * (-1)^u)
                if j < len(J):
                    ref = c0 * J[j][u] / div
                else:
                    ref = c0 * J[P - 1 - j][u] * (-1) ** u / div
                for i in range(P):
                    assert abs(v[0][i][j] - ref) < tol * c0, (k, u, i, j, v[0][i][j], ref)


def test_fdct_idct_roundtrip(oracle_mod):
    # FDCT (scipy dctn, = T.81 A.3.3 FDCT) of integer-valued coefficients'
    # reconstruction recovers them.
    rng = np.random.default_rng(5)
    q = np.ones(64, np.uint16)
    blocks = rng.integers(-200, 201, size=(8, 64))
    v, _ = _v_blocks(oracle_mod, _plane_of_blocks(blocks), q, 1)
    for b in range(8):
        back = fft.dctn(v[b], norm="ortho").ravel()
        assert np.max(np.abs(back - blocks[b])) < 1e-9


def test_dequant_uses_table_per_index(oracle_mod):
    # D = coef * Q[k] element-wise in natural order: scale one coefficient.
    q = np.ones(64, np.uint16)
    q[9] = 7
    c = np.zeros(64, np.int16)
    c[9] = 3
    v7, _ = _v_blocks(oracle_mod, _plane_of_blocks([c]), q, 1)
    c2 = np.zeros(64, np.int16)
    c2[9] = 21
    v1, _ = _v_blocks(oracle_mod, _plane_of_blocks([c2]), np.ones(64, np.uint16), 1)
    assert np.max(np.abs(v7 - v1)) < 1e-12
