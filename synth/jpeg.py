"""Baseline JPEG *encoder* stand-in: quantized coefficient planes -> JFIF bytes.

Input generation only (the encoder side of SURVEY §8(f) N4): it turns the
``CoefImage`` planes that ``synth`` already produces into a baseline
sequential-DCT JPEG file (ITU-T T.81 Annex B syntax, Huffman coding per
Annex F.1.2, restart intervals per B.2.4.4 / F.1.2.3), so the GPU Huffman
decoder and the CPU oracle's decoder can both start from the bytes a camera or
a web server would hand over.  It holds none of the decoder's arithmetic; the
oracle (``oracle/smol_oracle.c``) and the CUDA library each parse and decode
these bytes with their own code.

Huffman tables: the "typical" tables of T.81 Annex K.3 (Tables K.3-K.6), taken
from the DHT segments libjpeg writes (Pillow, ``optimize=False``), so no table
is retyped here.
"""
from __future__ import annotations

import functools
import io
import struct
from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np

from . import CoefImage

# T.81 Figure A.6: zig-zag sequence -> natural (row-major) index, generated
# by walking the anti-diagonals (even diagonals upwards, odd downwards).
def _zigzag() -> np.ndarray:
    order = []
    for s in range(15):
        cells = [(v, s - v) for v in range(8) if 0 <= s - v < 8]      # (row, col), row ascending
        if s % 2 == 0:
            cells.reverse()                                          # up-right: row descending
        order += [8 * v + u for v, u in cells]
    return np.array(order, dtype=np.int64)


ZIGZAG = _zigzag()


@functools.lru_cache(maxsize=1)
def standard_tables() -> Dict[Tuple[int, int], Tuple[bytes, bytes]]:
    """{(class, id): (BITS[16], HUFFVAL)} of T.81 Tables K.3 (DC luma), K.4
    (DC chroma), K.5 (AC luma), K.6 (AC chroma), read from libjpeg's output."""
    from PIL import Image
    buf = io.BytesIO()
    Image.new("RGB", (16, 16), (90, 140, 200)).save(buf, "JPEG", quality=75, optimize=False,
                                                     subsampling=2)
    b = buf.getvalue()
    out = {}
    i = 2
    while i < len(b) - 1:
        assert b[i] == 0xFF, "marker expected"
        m = b[i + 1]
        if m == 0xDA:
            break
        ln = struct.unpack(">H", b[i + 2:i + 4])[0]
        if m == 0xC4:
            j = i + 4
            while j < i + 2 + ln:
                tc_th = b[j]
                bits = bytes(b[j + 1:j + 17])
                nv = sum(bits)
                out[(tc_th >> 4, tc_th & 15)] = (bits, bytes(b[j + 17:j + 17 + nv]))
                j += 17 + nv
        i += 2 + ln
    assert set(out) == {(0, 0), (0, 1), (1, 0), (1, 1)}, out.keys()
    return out


def _codes(bits: bytes, vals: bytes) -> Dict[int, Tuple[int, int]]:
    """T.81 Annex C (Figures C.1-C.3): symbol -> (code, length)."""
    sizes = [l + 1 for l in range(16) for _ in range(bits[l])]
    code, k, table = 0, 0, {}
    si = sizes[0] if sizes else 0
    while k < len(sizes):
        while k < len(sizes) and sizes[k] == si:
            table[vals[k]] = (code, si)
            code += 1
            k += 1
        code <<= 1
        si += 1
    return table


class _BitWriter:
    """Entropy-coded segment writer with 0xFF byte stuffing (T.81 B.1.1.5)."""

    def __init__(self):
        self.out = bytearray()
        self.acc = 0
        self.n = 0

    def put(self, code: int, length: int):
        self.acc = (self.acc << length) | code
        self.n += length
        while self.n >= 8:
            self.n -= 8
            byte = (self.acc >> self.n) & 0xFF
            self.out.append(byte)
            if byte == 0xFF:
                self.out.append(0x00)
        self.acc &= (1 << self.n) - 1

    def align(self):
        """Pad to a byte boundary with 1-bits (T.81 F.1.2.3)."""
        if self.n:
            self.put((1 << (8 - self.n)) - 1, 8 - self.n)


def _category(v: int) -> int:
    return int(abs(v)).bit_length()


def _encode_block(w: _BitWriter, zz: np.ndarray, pred: int, dc_tab, ac_tab) -> int:
    """One block (zig-zag order, absolute DC): F.1.2.1 DC difference, F.1.2.2
    run-length AC with ZRL / EOB.  Returns the new DC predictor."""
    diff = int(zz[0]) - pred
    s = _category(diff)
    c, l = dc_tab[s]
    w.put(c, l)
    if s:
        w.put(diff if diff > 0 else diff + (1 << s) - 1, s)
    nz = np.flatnonzero(zz[1:]) + 1
    k = 1
    for kk in nz:
        r = int(kk) - k
        while r > 15:
            c, l = ac_tab[0xF0]            # ZRL
            w.put(c, l)
            r -= 16
        v = int(zz[kk])
        s = _category(v)
        c, l = ac_tab[(r << 4) | s]
        w.put(c, l)
        w.put(v if v > 0 else v + (1 << s) - 1, s)
        k = int(kk) + 1
    if k <= 63:
        c, l = ac_tab[0x00]                # EOB
        w.put(c, l)
    return int(zz[0])


def _sampling(img: CoefImage) -> List[Tuple[int, int]]:
    """(H, V) sampling factors per component (T.81 A.1.1)."""
    if img.gray:
        return [(1, 1)]
    hs, vs = {420: (2, 2), 422: (2, 1), 444: (1, 1)}[img.subsampling]
    return [(hs, vs), (1, 1), (1, 1)]


def encode(img: CoefImage, qtables: np.ndarray, restart_interval: int = 0) -> bytes:
    """Baseline JFIF file of ``img``'s coefficients.  ``restart_interval`` =
    MCUs per restart interval (T.81 B.2.4.4 DRI; 0 = none)."""
    tabs = standard_tables()
    hv = _sampling(img)
    nc = len(hv)
    hmax, vmax = max(h for h, _ in hv), max(v for _, v in hv)
    if nc == 1:                                  # non-interleaved: one block per MCU (A.2.2)
        mcux, mcuy = img.blocks_w[0], img.blocks_h[0]
    else:
        mcux, mcuy = -(-img.width // (8 * hmax)), -(-img.height // (8 * vmax))
        for c, (h, v) in enumerate(hv):
            assert img.blocks_w[c] >= mcux * h and img.blocks_h[c] >= mcuy * v, "planes not MCU-padded"
    tsel = [0] + [1] * (nc - 1)                  # luma tables 0, chroma tables 1
    qsel = list(img.qidx[:nc])
    zz = [np.asarray(p, dtype=np.int64).reshape(p.shape[0], p.shape[1], 64)[:, :, ZIGZAG] for p in img.coef]
    code = {(cl, t): _codes(*tabs[(cl, t)]) for cl in (0, 1) for t in (0, 1)}

    b = bytearray(b"\xFF\xD8")
    b += b"\xFF\xE0" + struct.pack(">H5sBBBHHBB", 16, b"JFIF\0", 1, 1, 0, 1, 1, 0, 0)
    for t in sorted(set(qsel)):                  # DQT, 8-bit, zig-zag order (B.2.4.1)
        b += b"\xFF\xDB" + struct.pack(">HB", 67, t) + bytes(int(x) for x in np.asarray(qtables[t])[ZIGZAG])
    b += b"\xFF\xC0" + struct.pack(">HBHHB", 8 + 3 * nc, 8, img.height, img.width, nc)   # SOF0
    for c in range(nc):
        b += struct.pack(">BBB", c + 1, (hv[c][0] << 4) | hv[c][1], qsel[c])
    for cl in (0, 1):                            # DHT (B.2.4.2)
        for t in sorted(set(tsel)):
            bits, vals = tabs[(cl, t)]
            b += b"\xFF\xC4" + struct.pack(">HB", 3 + 16 + len(vals), (cl << 4) | t) + bits + vals
    if restart_interval:
        b += b"\xFF\xDD" + struct.pack(">HH", 4, restart_interval)
    b += b"\xFF\xDA" + struct.pack(">HB", 6 + 2 * nc, nc)          # SOS
    for c in range(nc):
        b += struct.pack(">BB", c + 1, (tsel[c] << 4) | tsel[c])
    b += bytes([0, 63, 0])

    w = _BitWriter()
    pred = [0] * nc
    nmcu = mcux * mcuy
    for m in range(nmcu):
        if restart_interval and m and m % restart_interval == 0:
            w.align()
            b += w.out
            w.out = bytearray()
            b += bytes([0xFF, 0xD0 + ((m // restart_interval - 1) & 7)])   # RSTm
            pred = [0] * nc
        my, mx = divmod(m, mcux)
        for c in range(nc):
            h, v = hv[c] if nc > 1 else (1, 1)
            for y in range(v):
                for x in range(h):
                    pred[c] = _encode_block(w, zz[c][my * v + y, mx * h + x], pred[c],
                                            code[(0, tsel[c])], code[(1, tsel[c])])
    w.align()
    b += w.out
    b += b"\xFF\xD9"
    return bytes(b)


def encode_batch(imgs: Sequence[CoefImage], qtables: np.ndarray, restart_interval: int = 0
                 ) -> List[bytes]:
    """Encode a batch; repeated image objects (``batch_images`` replicates
    distinct images) are encoded once."""
    cache: Dict[int, bytes] = {}
    out = []
    for im in imgs:
        k = id(im)
        if k not in cache:
            cache[k] = encode(im, qtables, restart_interval)
        out.append(cache[k])
    return out
