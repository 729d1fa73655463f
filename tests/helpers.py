"""Test-side helpers: oracle references and the reading-R3 tie band.

Only calls oracle/ (and synth/); never the CUDA path.  Tie-free corpora are
built here (not in synth, which holds no decoder arithmetic) by rejecting
blocks whose oracle samples lie within delta_b of a rounding tie.
"""
from __future__ import annotations

import numpy as np

import oracle
import synth


def block_delta(coef: np.ndarray, q: np.ndarray) -> np.ndarray:
    """Reading R3 tie band per block: delta_b = max(2^-12, 2^-23 * sum |D|).
    coef [bh][bw][64] -> [bh][bw]."""
    D = np.abs(coef.astype(np.int64) * q.astype(np.int64)).sum(axis=-1)
    return np.maximum(2.0 ** -12, 2.0 ** -23 * D)


def tie_distance(v: np.ndarray) -> np.ndarray:
    """Distance of v + 128 from the nearest half-integer (a rounding tie)."""
    x = v + 128.0
    return np.abs(x - (np.floor(x) + 0.5))


def exact_basis_mask(k: int, idct_def: int = 0) -> np.ndarray:
    """[64] bool: coefficient (v, u) whose basis entries at scale 1/k are all
    exact (0 or +-1 times a power of two): u and v in {0, 4} at scale 1
    (t(4, x) = +-1), {0} plus the vanishing frequencies under Definition A
    (R1), {0, N/2} under Definition B (R16, N = 8/k)."""
    if idct_def and k > 1:
        N = 8 // k
        ok = {0, N // 2} if N > 1 else {0}
        ok |= set(range(N, 8))                  # unused: zero basis
    elif k == 1:
        ok = {0, 4}
    else:
        ok = {0} | {u for u in range(1, 8) if (k * u) % 16 == 0 or all(
            (k * u * (2 * j + 1)) % 16 == 8 for j in range(8 // k))}
    return np.array([(v in ok) and (u in ok) for v in range(8) for u in range(8)])


def plane_band(coef, q, k, v, idct_def: int = 0):
    """Boolean [h][w], reading R3: the sample lies within delta_b of a
    rounding tie but not exactly on it -- or exactly on it in a block with a
    nonzero coefficient whose basis is irrational: such a tie is reached only
    by cancellation of irrational terms (e.g. D(0,1) = D(1,0) at mirrored
    positions), which fp32 evaluation cannot reproduce exactly.  Exact ties
    of blocks whose arithmetic is exact (DC, u = 4 / N/2 paths) must match."""
    P = 8 // k
    h, w = v.shape
    delta = block_delta(coef, q)
    dl = np.repeat(np.repeat(delta, P, axis=0), P, axis=1)[:h, :w]
    inexact = ((coef != 0) & ~exact_basis_mask(k, idct_def)).any(axis=-1)
    il = np.repeat(np.repeat(inexact, P, axis=0), P, axis=1)[:h, :w]
    d = tie_distance(v)
    return (d <= dl) & ((d > 0) | il)


def oracle_planes(p, im, qt):
    """[(v, u8, band_mask)] for Y, Cb, Cr at the params' scale."""
    res = []
    c2s = bool(getattr(p, "chroma_2s", 0)) and len(im.coef) == 3 and getattr(im, "subsampling", 420) == 420
    for ci, (v, u8) in enumerate(oracle.decode_image_planes(p, im, qt, with_v=True)):
        q = qt[im.qidx[ci]]
        k = p.scale_denom // 2 if (ci > 0 and c2s) else p.scale_denom     # reading R18
        res.append((v, u8, plane_band(im.coef[ci], q, k, v, p.idct_def)))
    return res


def make_tie_free(im, qt, k: int, max_iter: int = 50, idct_def: int = 0):
    """Perturb AC coefficients of blocks having a sample within delta_b of a
    tie (exact ties excluded as well) until none does, at decode scale 1/k
    (Definition A, or B with idct_def = 1: nudges stay in the top-left)."""
    P = 8 // k
    coef = [c.copy() for c in im.coef]
    rng = np.random.default_rng(12345)
    for ci in range(len(coef)):
        q = qt[im.qidx[ci]]
        bh, bw = coef[ci].shape[:2]
        for _ in range(max_iter):
            v, _ = oracle.decode_plane(coef[ci], q, k, bw * P, bh * P, idct_def)
            delta = block_delta(coef[ci], q)
            d = tie_distance(v).reshape(bh, P, bw, P).min(axis=(1, 3))
            bad = d <= delta
            if not bad.any():
                break
            idx = np.argwhere(bad)
            for (by, bx) in idx:
                # an odd-u AC nudge shifts samples by irrational amounts; at
                # scale 1/8 only the DC matters
                choices = [1, 8, 9] if (idct_def and k == 4) else [1, 3, 8, 24, 9]
                j = 0 if k == 8 else int(rng.choice(choices))
                coef[ci][by, bx, j] += 1 if rng.random() < 0.5 else -1
        else:
            raise RuntimeError("tie-free regeneration did not converge")
    return synth.CoefImage(im.width, im.height, coef, im.qidx, getattr(im, "subsampling", 420))


def rgb_from_planes(Y, Cb, Cr, subsampling=420):
    return oracle.upsample_color(Y, Cb, Cr, subsampling)[1]


def _taps(n_out, offset, n_in, n_res):
    """R8 taps (i0, i1) of output indices offset..offset+n_out-1 in exact ints."""
    d = np.arange(n_out, dtype=np.int64) + offset
    num = np.maximum(0, (2 * d + 1) * n_in - n_res)
    i0 = np.minimum(num // (2 * n_res), n_in - 1)
    i1 = np.minimum(i0 + 1, n_in - 1)
    return i0, i1


def affected_outputs(po, im, qt, roi=None):
    """Boolean [OH][OW]: outputs whose bilinear taps touch an RGB pixel that
    depends on a decoded sample inside the reading-R3 tie band (where the
    kernel may legitimately differ by one u8 level)."""
    g = oracle.geometry(po, im.width, im.height)
    left, top = (g.left, g.top) if roi is None else roi
    bands = [b for (_, _, b) in oracle_planes(po, im, qt)]
    pix = bands[0]
    if len(bands) == 3:
        c16, _ = oracle.upsample_color(np.zeros((g.Hd, g.Wd), np.uint8),
                                       bands[1].astype(np.uint8), bands[2].astype(np.uint8))
        pix = pix | (c16[..., 0] > 0) | (c16[..., 1] > 0)
    y0, y1 = _taps(g.OH, top, g.Hd, g.Hr)
    x0, x1 = _taps(g.OW, left, g.Wd, g.Wr)
    return (pix[y0][:, x0] | pix[y0][:, x1] | pix[y1][:, x0] | pix[y1][:, x1])
