"""Coefficient-block layouts of the C ABI (include/smol_preproc.h
smol_coef_layout) -- host-side packing of dense entropy-decoded planes.

PACKED keeps, per 8x8 block, only the coefficients whose box-averaged basis
a_k(u, .) is not identically zero at decode scale 1/k (reading R1), row-major
over the index set, padded to 8 bytes; block rows padded to 16 bytes.  A host
entropy decoder would write this format directly; here it is produced from
dense planes.  With the Definition B reduced-scale IDCT (reading R16) the
kept set is the top-left (8/k) x (8/k) coefficients (16 / 4 / 1 at k = 2 /
4 / 8), which need no padding.
"""
from __future__ import annotations

import numpy as np

_SETS = {1: list(range(8)), 2: [0, 1, 2, 3, 5, 6, 7], 4: [0, 1, 3, 5, 7], 8: [0]}


def block_elems(k: int, packed: bool = True, truncated: bool = False) -> int:
    """int16 elements per stored block (DENSE64: 64)."""
    if not packed or k == 1:
        return 64
    if truncated:
        return (8 // k) ** 2
    return {2: 52, 4: 28, 8: 1}[k]


def index_set(k: int, truncated: bool = False):
    """Natural-order coefficient indices (v*8+u) kept at scale 1/k."""
    s = list(range(8 // k)) if truncated else _SETS[k]
    return [v * 8 + u for v in s for u in s]


def pack_plane(coef: np.ndarray, k: int, truncated: bool = False) -> np.ndarray:
    """[bh][bw][64] int16 -> [bh][row_stride/2] int16 with 16-byte rows."""
    bh, bw, _ = coef.shape
    e = block_elems(k, True, truncated)
    if e == 64:
        return np.ascontiguousarray(coef, dtype=np.int16).reshape(bh, bw * 64)
    idx = index_set(k, truncated)
    row = -(-(bw * e * 2) // 16) * 16 // 2          # elements per padded row
    out = np.zeros((bh, row), np.int16)
    blk = np.zeros((bh, bw, e), np.int16)
    blk[:, :, :len(idx)] = coef[:, :, idx]
    out[:, :bw * e] = blk.reshape(bh, bw * e)
    return out
