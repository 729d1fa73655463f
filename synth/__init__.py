"""Seeded synthetic inputs for the Smol preprocessing hot path.

This module is the ONLY code shared by the CUDA path's tests/bench and the CPU
oracle's tests.  It holds none of the method's (decoder-side) arithmetic: it
plays the role of the *encoder* plus the host entropy decoder (SURVEY §8(a)
row a0: "Huffman decode -> quantized coefficients, DC prediction undone").
It produces what a baseline JPEG decoder hands to the GPU after entropy
decoding: per component, int16 quantized DCT coefficients in natural
(row-major) order, block-raster layout ``[blocks_h][blocks_w][64]`` with
absolute DC, plus uint16 quantization tables in natural order.

Workload shapes follow BASELINE.json ``configs`` (c1..c5, see CONFIGS) and the
paper's workloads: ImageNet-shaped 500x375 JPEGs (§2 ResNet
preprocessing), 161x161 thumbnails (§5.2), 1080p video frames
(P:1271-1274).  Quality 75 / 95 follow P:1307-1308.

Recipes (restated in DESIGN.md §Inputs):
  natural : smooth multi-octave random RGB field + fine texture on ~60% of
            the area + 4 hard-edged rectangles, clipped to u8; JFIF forward
            colour transform; 2x2-mean chroma downsample (4:2:0); edge
            replicate to 16x16 MCU multiples; level shift -128; orthonormal
            8x8 FDCT (= T.81 A.3.3 FDCT); quantize with IJG-scaled Annex K
            tables, round half away from zero.
  stress  : dense uniform coefficients with dequantized |D| <= 2047 (the valid
            8-bit baseline range), plus 5% DC-only blocks and 2% saturating
            blocks.
"""
from __future__ import annotations

import dataclasses
from typing import List, Optional, Sequence, Tuple

import numpy as np

SEED_BASE = 2007_13005

# T.81 Annex K, Table K.1 (luminance) and K.2 (chrominance), natural order.
ANNEX_K1 = np.array([
    16, 11, 10, 16, 24, 40, 51, 61,
    12, 12, 14, 19, 26, 58, 60, 55,
    14, 13, 16, 24, 40, 57, 69, 56,
    14, 17, 22, 29, 51, 87, 80, 62,
    18, 22, 37, 56, 68, 109, 103, 77,
    24, 35, 55, 64, 81, 104, 113, 92,
    49, 64, 78, 87, 103, 121, 120, 101,
    72, 92, 95, 98, 112, 100, 103, 99], dtype=np.int64)
ANNEX_K2 = np.array([
    17, 18, 24, 47, 99, 99, 99, 99,
    18, 21, 26, 66, 99, 99, 99, 99,
    24, 26, 56, 99, 99, 99, 99, 99,
    47, 66, 99, 99, 99, 99, 99, 99,
    99, 99, 99, 99, 99, 99, 99, 99,
    99, 99, 99, 99, 99, 99, 99, 99,
    99, 99, 99, 99, 99, 99, 99, 99,
    99, 99, 99, 99, 99, 99, 99, 99], dtype=np.int64)

# ImageNet normalisation constants (torchvision convention), RGB order.
IMAGENET_MEAN = (0.485, 0.456, 0.406)
IMAGENET_STD = (0.229, 0.224, 0.225)


def ijg_quant_table(base: np.ndarray, quality: int) -> np.ndarray:
    """IJG quality scaling of an Annex K table (libjpeg jcparam.c convention)."""
    quality = int(min(max(quality, 1), 100))
    scale = 5000 // quality if quality < 50 else 200 - 2 * quality
    q = (base * scale + 50) // 100
    return np.clip(q, 1, 255).astype(np.uint16)


def quant_tables(quality: int) -> np.ndarray:
    """[2][64] uint16: table 0 = luma, table 1 = chroma."""
    return np.stack([ijg_quant_table(ANNEX_K1, quality),
                     ijg_quant_table(ANNEX_K2, quality)])


@dataclasses.dataclass
class CoefImage:
    """One entropy-decoded JPEG: 3 coefficient planes [bh][bw][64] int16
    (4:2:0 Y, Cb, Cr) or 1 (grayscale Y)."""
    width: int
    height: int
    coef: List[np.ndarray]                 # Y, Cb, Cr  (or Y only)
    qidx: Tuple[int, ...] = (0, 1, 1)
    subsampling: int = 420                 # 420, 422, 444 (chroma W/hs x H/vs), or 400 (gray)

    @property
    def gray(self) -> bool:
        return len(self.coef) == 1

    @property
    def blocks_w(self):
        return [c.shape[1] for c in self.coef]

    @property
    def blocks_h(self):
        return [c.shape[0] for c in self.coef]

    def nbytes(self) -> int:
        return sum(c.nbytes for c in self.coef)


@dataclasses.dataclass
class Config:
    name: str
    n: int
    width: int
    height: int
    scale_denom: int
    resize_mode: str          # "short" | "exact"
    resize_short: int = 0
    resize_w: int = 0
    resize_h: int = 0
    crop_w: int = 0
    crop_h: int = 0
    out_dtype: str = "f32"    # "f32" | "f16"
    quality: int = 75
    index: int = 0

    @property
    def out_hw(self) -> Tuple[int, int]:
        if self.crop_w:
            return self.crop_h, self.crop_w
        if self.resize_mode == "exact":
            return self.resize_h, self.resize_w
        raise ValueError("short-side resize without crop has image-dependent size")


# BASELINE.json "configs" (index 1..5).  c3 is split by decode scale.
CONFIGS = {
    "c1": Config("c1", 8, 64, 64, 1, "exact", resize_w=32, resize_h=32, index=1),
    "c2": Config("c2", 256, 500, 375, 1, "short", resize_short=256, crop_w=224, crop_h=224, index=2),
    "c3a": Config("c3a", 256, 500, 375, 2, "short", resize_short=256, crop_w=224, crop_h=224,
                  out_dtype="f16", index=3),
    "c3b": Config("c3b", 256, 500, 375, 4, "short", resize_short=256, crop_w=224, crop_h=224,
                  out_dtype="f16", index=3),
    "c4": Config("c4", 4096, 161, 161, 8, "exact", resize_w=64, resize_h=64, index=4),
    "c5": Config("c5", 1024, 1920, 1080, 4, "exact", resize_w=224, resize_h=224, index=5),
}


# ----------------------------------------------------------------- images ---

def _cubic_matrix(n_out: int, n_grid: int, cell: float, offset: float) -> np.ndarray:
    """[n_out][n_grid] Catmull-Rom interpolation weights sampling a grid of
    spacing ``cell`` px at positions offset + i."""
    pos = (np.arange(n_out) + offset) / cell + 1.0
    i0 = np.floor(pos).astype(np.int64)
    t = pos - i0
    w = np.stack([(-t ** 3 + 2 * t ** 2 - t) / 2, (3 * t ** 3 - 5 * t ** 2 + 2) / 2,
                  (-3 * t ** 3 + 4 * t ** 2 + t) / 2, (t ** 3 - t ** 2) / 2], axis=1)
    m = np.zeros((n_out, n_grid))
    for k in range(4):
        np.add.at(m, (np.arange(n_out), np.clip(i0 - 1 + k, 0, n_grid - 1)), w[:, k])
    return m


def _smooth_field(rng: np.random.Generator, h: int, w: int, cell: float) -> np.ndarray:
    """Unit-variance smooth random field: random grid with spacing ``cell`` px,
    Catmull-Rom upsampled (separable matrices)."""
    gh = int(np.ceil(h / cell)) + 4
    gw = int(np.ceil(w / cell)) + 4
    g = rng.standard_normal((gh, gw))
    f = _cubic_matrix(h, gh, cell, rng.random() * cell) @ g @ _cubic_matrix(w, gw, cell, rng.random() * cell).T
    s = f.std()
    return (f - f.mean()) / (s if s > 0 else 1.0)


def natural_rgb(rng: np.random.Generator, width: int, height: int) -> np.ndarray:
    """[H][W][3] uint8 photo-like test image (smooth regions, texture, edges)."""
    h, w = height, width
    big = max(4.0, min(h, w) / 4.0)
    mid = max(3.0, min(h, w) / 12.0)
    lum = 128 + 55 * _smooth_field(rng, h, w, big) + 25 * _smooth_field(rng, h, w, mid)
    # texture only where a smooth mask is positive (~60% of the area)
    mask = np.clip(_smooth_field(rng, h, w, big) + 0.25, 0, 1)
    tex = rng.standard_normal((h, w))
    tex = 0.5 * tex + 0.25 * (np.roll(tex, 1, 0) + np.roll(tex, 1, 1))   # mildly low-passed
    lum = lum + 7 * mask * tex
    rgb = np.empty((h, w, 3))
    for c in range(3):
        rgb[..., c] = lum + 30 * _smooth_field(rng, h, w, big) + 8 * _smooth_field(rng, h, w, mid)
    for _ in range(4):                           # hard-edged rectangles
        y0, x0 = rng.integers(0, h), rng.integers(0, w)
        y1 = min(h, y0 + rng.integers(1, max(2, h // 3)))
        x1 = min(w, x0 + rng.integers(1, max(2, w // 3)))
        rgb[y0:y1, x0:x1, :] += rng.normal(0, 40, size=3)
    return np.clip(np.rint(rgb), 0, 255).astype(np.uint8)


def _rgb_to_ycbcr(rgb: np.ndarray) -> np.ndarray:
    """JFIF 1.02 forward transform (encoder side)."""
    r, g, b = (rgb[..., i].astype(np.float64) for i in range(3))
    y = 0.299 * r + 0.587 * g + 0.114 * b
    cb = -0.168736 * r - 0.331264 * g + 0.5 * b + 128.0
    cr = 0.5 * r - 0.418688 * g - 0.081312 * b + 128.0
    return np.stack([y, cb, cr], axis=-1)


def _pad_edge(plane: np.ndarray, ph: int, pw: int) -> np.ndarray:
    h, w = plane.shape
    return np.pad(plane, ((0, ph - h), (0, pw - w)), mode="edge")


def _fdct_quantize(plane: np.ndarray, q: np.ndarray) -> np.ndarray:
    """Blocks of an (already padded) plane -> [bh][bw][64] int16 (encoder)."""
    from scipy import fft
    h, w = plane.shape
    bh, bw = h // 8, w // 8
    blocks = (plane - 128.0).reshape(bh, 8, bw, 8).transpose(0, 2, 1, 3)
    S = fft.dctn(blocks, type=2, norm="ortho", axes=(-2, -1)).reshape(bh, bw, 64)
    qv = q.astype(np.float64)
    t = S / qv
    c = np.sign(t) * np.floor(np.abs(t) + 0.5)          # round half away from zero
    return np.clip(c, -32768, 32767).astype(np.int16)


def encode_420(rgb: np.ndarray, qtables: np.ndarray) -> CoefImage:
    """Encoder stand-in: u8 RGB -> entropy-decoded 4:2:0 coefficient planes."""
    h, w, _ = rgb.shape
    ycc = _rgb_to_ycbcr(rgb)
    mh, mw = -(-h // 16), -(-w // 16)                    # MCU grid
    Y = _pad_edge(ycc[..., 0], 16 * mh, 16 * mw)
    ch, cw = -(-h // 2), -(-w // 2)
    planes = [Y]
    for ci in (1, 2):
        c = _pad_edge(ycc[..., ci], 2 * ch, 2 * cw)
        c = c.reshape(ch, 2, cw, 2).mean(axis=(1, 3))     # 2x2 mean downsample
        planes.append(_pad_edge(c, 8 * mh, 8 * mw))
    coef = [_fdct_quantize(planes[0], qtables[0]),
            _fdct_quantize(planes[1], qtables[1]),
            _fdct_quantize(planes[2], qtables[1])]
    return CoefImage(w, h, coef)


# chroma subsampling factors (hs, vs) per T.81 A.1.1 (Hmax/Hc, Vmax/Vc)
SUBSAMPLING = {420: (2, 2), 422: (2, 1), 444: (1, 1)}


def encode_ycc(rgb: np.ndarray, qtables: np.ndarray, subsampling: int = 420) -> CoefImage:
    """Encoder stand-in for any of the 3-component samplings: JFIF forward
    transform, hs x vs mean chroma downsample, MCU (8 hs x 8 vs luma px)
    edge padding, FDCT + quantize."""
    if subsampling == 420:
        return encode_420(rgb, qtables)
    hs, vs = SUBSAMPLING[subsampling]
    h, w, _ = rgb.shape
    ycc = _rgb_to_ycbcr(rgb)
    mh, mw = -(-h // (8 * vs)), -(-w // (8 * hs))           # MCU grid
    planes = [_pad_edge(ycc[..., 0], 8 * vs * mh, 8 * hs * mw)]
    ch, cw = -(-h // vs), -(-w // hs)
    for ci in (1, 2):
        c = _pad_edge(ycc[..., ci], vs * ch, hs * cw)
        c = c.reshape(ch, vs, cw, hs).mean(axis=(1, 3))     # hs x vs mean downsample
        planes.append(_pad_edge(c, 8 * mh, 8 * mw))
    coef = [_fdct_quantize(planes[0], qtables[0]),
            _fdct_quantize(planes[1], qtables[1]),
            _fdct_quantize(planes[2], qtables[1])]
    return CoefImage(w, h, coef, subsampling=subsampling)


def encode_gray(rgb: np.ndarray, qtables: np.ndarray) -> CoefImage:
    """Encoder stand-in for a grayscale JPEG: JFIF luma of the RGB field, one
    component, 8x8 MCUs (T.81 A.2.2: non-interleaved single component)."""
    h, w, _ = rgb.shape
    Y = _rgb_to_ycbcr(rgb)[..., 0]
    Y = _pad_edge(Y, 8 * -(-h // 8), 8 * -(-w // 8))
    return CoefImage(w, h, [_fdct_quantize(Y, qtables[0])], (0,), subsampling=400)


def stress_image(rng: np.random.Generator, width: int, height: int,
                 qtables: np.ndarray, limit: int = 2047) -> CoefImage:
    """Dense uniform coefficients with dequantized |D| <= limit, plus 5% DC-only
    and 2% saturating blocks."""
    mh, mw = -(-height // 16), -(-width // 16)
    coef = []
    for ci, (bh, bw) in enumerate([(2 * mh, 2 * mw), (mh, mw), (mh, mw)]):
        q = qtables[0 if ci == 0 else 1].astype(np.int64)
        lim = limit // q
        c = rng.integers(-lim, lim + 1, size=(bh, bw, 64))
        u = rng.random((bh, bw))
        dc_only = u < 0.05
        c[dc_only, 1:] = 0
        sat = (u >= 0.05) & (u < 0.07)
        c[sat, 1:] = 0
        c[sat, 0] = np.where(rng.random(int(sat.sum())) < 0.5, lim[0], -lim[0])
        coef.append(c.astype(np.int16))
    return CoefImage(width, height, coef)


def make_image(rng: np.random.Generator, width: int, height: int, qtables: np.ndarray,
               mode: str = "natural") -> CoefImage:
    if mode == "natural":
        return encode_420(natural_rgb(rng, width, height), qtables)
    if mode == "stress":
        return stress_image(rng, width, height, qtables)
    if mode == "gray":
        return encode_gray(natural_rgb(rng, width, height), qtables)
    if mode in ("natural422", "natural444"):
        return encode_ycc(natural_rgb(rng, width, height), qtables, int(mode[-3:]))
    raise ValueError(mode)


def distinct_images(cfg: Config, mode: str = "natural", quality: Optional[int] = None,
                    n_distinct: Optional[int] = None, seed_offset: int = 0
                    ) -> Tuple[List[CoefImage], np.ndarray]:
    """``min(N, 64)`` distinct seeded images of ``cfg``'s shape + qtables."""
    q = cfg.quality if quality is None else quality
    qt = quant_tables(q)
    nd = min(cfg.n, 64) if n_distinct is None else n_distinct
    ss = np.random.SeedSequence(SEED_BASE + cfg.index + 1000 * seed_offset)
    rngs = [np.random.default_rng(s) for s in ss.spawn(nd)]
    if nd >= 4 and cfg.width * cfg.height >= 1 << 18:
        # large frames: one thread per image (each has its own generator, so
        # the result does not depend on the thread count)
        import os
        from concurrent.futures import ThreadPoolExecutor
        with ThreadPoolExecutor(min(nd, os.cpu_count() or 1)) as ex:
            return list(ex.map(lambda r: make_image(r, cfg.width, cfg.height, qt, mode), rngs)), qt
    return [make_image(r, cfg.width, cfg.height, qt, mode) for r in rngs], qt


def batch_images(cfg: Config, mode: str = "natural", quality: Optional[int] = None,
                 n: Optional[int] = None, n_distinct: Optional[int] = None
                 ) -> Tuple[List[CoefImage], np.ndarray]:
    """N images (distinct ones replicated) for config ``cfg``."""
    n = cfg.n if n is None else n
    imgs, qt = distinct_images(cfg, mode, quality, n_distinct=min(n, 64) if n_distinct is None else n_distinct)
    return [imgs[i % len(imgs)] for i in range(n)], qt


def random_sizes(rng: np.random.Generator, n: int, lo: int = 8, hi: int = 200
                 ) -> List[Tuple[int, int]]:
    return [(int(rng.integers(lo, hi)), int(rng.integers(lo, hi))) for _ in range(n)]


def coef_stats(imgs: Sequence[CoefImage]) -> dict:
    """Non-zeros per block and DC-only share per component class (reported
    with every benchmark)."""
    out = {}
    for name, sel in (("luma", [0]), ("chroma", [1, 2])):
        nz, dco, nb = 0, 0, 0
        for im in imgs:
            for ci in sel:
                c = im.coef[ci].reshape(-1, 64)
                nzc = (c != 0).sum(axis=1)
                nz += int(nzc.sum())
                dco += int(((c[:, 1:] != 0).sum(axis=1) == 0).sum())
                nb += c.shape[0]
        out[name] = {"nonzeros_per_block": nz / max(nb, 1), "dc_only_share": dco / max(nb, 1)}
    return out
