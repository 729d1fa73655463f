"""CPU oracle for the Smol preprocessing hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` legs may import this package.  The product path
(``paper_2007_13005_b200``) never imports it, and it imports nothing from the
product path: the two share only the seeded input generator (``synth``).

The arithmetic lives in plain C (``smol_oracle.c``, fp64, direct formulas);
this module is ctypes marshalling plus numpy containers.  See
``smol_oracle.h`` for what each function follows in the paper.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from concurrent.futures import ThreadPoolExecutor
from typing import Optional, Sequence, Tuple

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "smol_oracle.c")
_SRC_JPEG = os.path.join(_HERE, "smol_oracle_jpeg.c")
_LIB_PATH = os.path.join(_HERE, "libsmol_oracle.so")
_lib = None


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (plain -O2, no -ffast-math)."""
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < max(
            os.path.getmtime(_SRC), os.path.getmtime(_SRC_JPEG),
            os.path.getmtime(os.path.join(_HERE, "smol_oracle.h"))):
        tmp = _LIB_PATH + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-std=c99", "-Wall", "-fPIC", "-shared",
                               "-fno-fast-math", "-o", tmp, _SRC, _SRC_JPEG, "-lm"])
        os.replace(tmp, _LIB_PATH)
    return _LIB_PATH


class _Plane(ctypes.Structure):
    _fields_ = [("coef", ctypes.c_void_p), ("blocks_w", ctypes.c_int32),
                ("blocks_h", ctypes.c_int32), ("row_stride", ctypes.c_int32),
                ("q", ctypes.c_void_p)]


class _Image(ctypes.Structure):
    _fields_ = [("width", ctypes.c_int32), ("height", ctypes.c_int32), ("comp", _Plane * 3),
                ("hs", ctypes.c_int32), ("vs", ctypes.c_int32)]


class _Params(ctypes.Structure):
    _fields_ = [("scale_denom", ctypes.c_int32), ("resize_mode", ctypes.c_int32),
                ("resize_short", ctypes.c_int32), ("resize_w", ctypes.c_int32),
                ("resize_h", ctypes.c_int32), ("crop_w", ctypes.c_int32),
                ("crop_h", ctypes.c_int32), ("mean", ctypes.c_double * 3),
                ("std", ctypes.c_double * 3), ("out_f16", ctypes.c_int32),
                ("idct_def", ctypes.c_int32), ("chroma_2s", ctypes.c_int32)]


class Geometry(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int32) for n in
                ("Wd", "Hd", "Wc", "Hc", "Wr", "Hr", "left", "top", "OW", "OH")]

    def as_dict(self):
        return {n: getattr(self, n) for n, _ in self._fields_}


def lib():
    global _lib
    if _lib is None:
        L = ctypes.CDLL(build())
        P = ctypes.POINTER
        L.oracle_geometry_of.argtypes = [P(_Params), ctypes.c_int32, ctypes.c_int32, P(Geometry)]
        L.oracle_geometry_of2.argtypes = [P(_Params), ctypes.c_int32, ctypes.c_int32, ctypes.c_int32,
                                          ctypes.c_int32, P(Geometry)]
        L.oracle_decode_plane.argtypes = [P(_Plane), ctypes.c_int32, ctypes.c_int32, ctypes.c_int32,
                                          ctypes.c_void_p, ctypes.c_void_p]
        L.oracle_decode_plane2.argtypes = [P(_Plane), ctypes.c_int32, ctypes.c_int32, ctypes.c_int32,
                                           ctypes.c_int32, ctypes.c_void_p, ctypes.c_void_p]
        L.oracle_upsample_color2.argtypes = [ctypes.c_void_p, ctypes.c_int32, ctypes.c_int32,
                                             ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int32,
                                             ctypes.c_int32, ctypes.c_int32, ctypes.c_int32,
                                             ctypes.c_void_p, ctypes.c_void_p]
        L.oracle_run_image2.argtypes = [P(_Params), P(_Image)] + [ctypes.c_int32] * 6 + [ctypes.c_void_p]
        L.oracle_upsample_color.argtypes = [ctypes.c_void_p, ctypes.c_int32, ctypes.c_int32,
                                            ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int32,
                                            ctypes.c_int32, ctypes.c_void_p, ctypes.c_void_p]
        L.oracle_color.argtypes = [ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, ctypes.c_void_p]
        L.oracle_color.restype = None
        L.oracle_resize_crop_normalize.argtypes = (
            [ctypes.c_void_p] + [ctypes.c_int32] * 8 + [ctypes.c_void_p, ctypes.c_void_p,
                                                        ctypes.c_int32, ctypes.c_void_p,
                                                        ctypes.c_void_p])
        L.oracle_run_image.argtypes = [P(_Params), P(_Image), ctypes.c_int32, ctypes.c_int32,
                                       ctypes.c_void_p]
        L.oracle_alg1_crop_window.argtypes = [ctypes.c_int32] * 3 + [P(ctypes.c_int32)] * 4
        L.oracle_f64_to_f16.argtypes = [ctypes.c_double]
        L.oracle_jpeg_info_of.argtypes = [ctypes.c_char_p, ctypes.c_int64, P(JpegInfo)]
        L.oracle_jpeg_decode.argtypes = [ctypes.c_char_p, ctypes.c_int64, ctypes.c_void_p * 3]
        L.oracle_f64_to_f16.restype = ctypes.c_uint16
        _lib = L
    return _lib


def _ptr(a: np.ndarray) -> int:
    assert a.flags["C_CONTIGUOUS"]
    return a.ctypes.data


def make_params(scale_denom=1, resize_mode="short", resize_short=256, resize_w=0, resize_h=0,
                crop_w=0, crop_h=0, mean=(0.485, 0.456, 0.406), std=(0.229, 0.224, 0.225),
                out_dtype="f32", idct_def="box", chroma_2s=False) -> _Params:
    p = _Params()
    p.scale_denom = scale_denom
    p.resize_mode = 0 if resize_mode == "short" else 1
    p.resize_short, p.resize_w, p.resize_h = resize_short, resize_w, resize_h
    p.crop_w, p.crop_h = crop_w, crop_h
    p.mean = (ctypes.c_double * 3)(*mean)
    p.std = (ctypes.c_double * 3)(*std)
    p.out_f16 = 1 if out_dtype == "f16" else 0
    p.idct_def = 1 if idct_def == "truncated" else 0
    p.chroma_2s = 1 if chroma_2s else 0
    return p


def params_from_config(cfg, mean=None, std=None, idct_def="box", chroma_2s=False) -> _Params:
    kw = {"idct_def": idct_def, "chroma_2s": chroma_2s}
    if mean is not None:
        kw["mean"] = mean
    if std is not None:
        kw["std"] = std
    return make_params(cfg.scale_denom, cfg.resize_mode, cfg.resize_short, cfg.resize_w,
                       cfg.resize_h, cfg.crop_w, cfg.crop_h, out_dtype=cfg.out_dtype, **kw)


SUBSAMPLING = {420: (2, 2), 422: (2, 1), 444: (1, 1), 400: (2, 2)}


def geometry(p: _Params, width: int, height: int, subsampling: int = 420) -> Geometry:
    g = Geometry()
    hs, vs = SUBSAMPLING[subsampling]
    rc = lib().oracle_geometry_of2(ctypes.byref(p), width, height, hs, vs, ctypes.byref(g))
    if rc:
        raise ValueError(f"oracle_geometry_of failed rc={rc}")
    return g


def _plane(coef: np.ndarray, q: np.ndarray) -> _Plane:
    pl = _Plane()
    pl.coef = _ptr(coef)
    pl.blocks_h, pl.blocks_w = coef.shape[0], coef.shape[1]
    pl.row_stride = coef.shape[1] * 64
    pl.q = _ptr(q)
    return pl


def decode_plane(coef: np.ndarray, q: np.ndarray, k: int, out_w: int, out_h: int, idct_def: int = 0
                 ) -> Tuple[np.ndarray, np.ndarray]:
    """-> (v [out_h][out_w] f64 before level shift, u8 [out_h][out_w]);
    idct_def 0 = Definition A (R1), 1 = Definition B (R16)."""
    coef = np.ascontiguousarray(coef, dtype=np.int16)
    q = np.ascontiguousarray(q, dtype=np.uint16)
    v = np.empty((out_h, out_w), np.float64)
    u8 = np.empty((out_h, out_w), np.uint8)
    pl = _plane(coef, q)
    rc = lib().oracle_decode_plane2(ctypes.byref(pl), k, idct_def, out_w, out_h, _ptr(v), _ptr(u8))
    if rc:
        raise ValueError(f"oracle_decode_plane rc={rc}")
    return v, u8


def upsample_color(Y: np.ndarray, Cb: np.ndarray, Cr: np.ndarray, subsampling: int = 420
                   ) -> Tuple[np.ndarray, np.ndarray]:
    """-> (c16 [Hd][Wd][2] int32, rgb [Hd][Wd][3] u8)."""
    hs, vs = SUBSAMPLING[subsampling]
    Y, Cb, Cr = (np.ascontiguousarray(a, dtype=np.uint8) for a in (Y, Cb, Cr))
    Hd, Wd = Y.shape
    Hc, Wc = Cb.shape
    c16 = np.empty((Hd, Wd, 2), np.int32)
    rgb = np.empty((Hd, Wd, 3), np.uint8)
    rc = lib().oracle_upsample_color2(_ptr(Y), Wd, Hd, _ptr(Cb), _ptr(Cr), Wc, Hc, hs, vs, _ptr(c16),
                                      _ptr(rgb))
    if rc:
        raise ValueError(f"oracle_upsample_color rc={rc}")
    return c16, rgb


def color(Y: int, cb16: int, cr16: int) -> Tuple[int, int, int]:
    out = (ctypes.c_uint8 * 3)()
    lib().oracle_color(Y, cb16, cr16, out)
    return tuple(out)


def resize_crop_normalize(rgb: np.ndarray, Wr: int, Hr: int, left: int, top: int, OW: int, OH: int,
                          mean=(0.485, 0.456, 0.406), std=(0.229, 0.224, 0.225), out_dtype="f32"
                          ) -> Tuple[np.ndarray, np.ndarray]:
    """-> (out [3][OH][OW] f32/f16, resized-before-normalize [3][OH][OW] f64)."""
    rgb = np.ascontiguousarray(rgb, dtype=np.uint8)
    Hd, Wd, _ = rgb.shape
    out = np.empty((3, OH, OW), np.float16 if out_dtype == "f16" else np.float32)
    res = np.empty((3, OH, OW), np.float64)
    m = (ctypes.c_double * 3)(*mean)
    s = (ctypes.c_double * 3)(*std)
    rc = lib().oracle_resize_crop_normalize(_ptr(rgb), Wd, Hd, Wr, Hr, left, top, OW, OH, m, s,
                                            1 if out_dtype == "f16" else 0, _ptr(out), _ptr(res))
    if rc:
        raise ValueError(f"oracle_resize_crop_normalize rc={rc}")
    return out, res


def _image(im, qtables: np.ndarray, keep: list) -> _Image:
    c = _Image()
    c.width, c.height = im.width, im.height
    c.hs, c.vs = SUBSAMPLING[getattr(im, "subsampling", 420)]
    for ci in range(3):
        if ci >= len(im.coef):               # grayscale: one component
            c.comp[ci] = _Plane()
            continue
        coef = np.ascontiguousarray(im.coef[ci], dtype=np.int16)
        q = np.ascontiguousarray(qtables[im.qidx[ci]], dtype=np.uint16)
        keep += [coef, q]
        c.comp[ci] = _plane(coef, q)
    return c


def run_image(p: _Params, im, qtables: np.ndarray, roi: Optional[Tuple[int, int]] = None,
              roi_rect: Optional[Tuple[int, int, int, int]] = None) -> np.ndarray:
    """Whole pipeline for one synth.CoefImage -> [3][OH][OW] (f32 or f16).
    roi: crop-window origin in resized coordinates; roi_rect: (x, y, w, h) ROI
    rectangle in SOF pixels, resized to the plan's output size (R15)."""
    g = geometry(p, im.width, im.height, getattr(im, "subsampling", 420))
    keep: list = []
    c = _image(im, qtables, keep)
    OW, OH = g.OW, g.OH
    if roi_rect is not None:
        OW = p.crop_w if p.crop_w > 0 else p.resize_w
        OH = p.crop_h if p.crop_w > 0 else p.resize_h
    out = np.empty((3, OH, OW), np.float16 if p.out_f16 else np.float32)
    left, top = roi if roi is not None else (-1, -1)
    rx, ry, rw, rh = roi_rect if roi_rect is not None else (0, 0, 0, 0)
    rc = lib().oracle_run_image2(ctypes.byref(p), ctypes.byref(c), left, top, rx, ry, rw, rh, _ptr(out))
    if rc:
        raise ValueError(f"oracle_run_image rc={rc}")
    return out


def run_batch(p: _Params, imgs: Sequence, qtables: np.ndarray, threads: int = 1,
              rois: Optional[Sequence] = None) -> np.ndarray:
    """Pipeline over a batch (thread pool over images; ctypes drops the GIL)."""
    rois = rois if rois is not None else [None] * len(imgs)
    if threads <= 1:
        outs = [run_image(p, im, qtables, r) for im, r in zip(imgs, rois)]
    else:
        with ThreadPoolExecutor(threads) as ex:
            outs = list(ex.map(lambda a: run_image(p, a[0], qtables, a[1]), zip(imgs, rois)))
    return np.stack(outs)


def decode_image_planes(p: _Params, im, qtables: np.ndarray, with_v: bool = False):
    """Decoded u8 Y, Cb, Cr planes (Y only for a grayscale image) and optional
    unrounded v at p's scale."""
    g = geometry(p, im.width, im.height, getattr(im, "subsampling", 420))
    k = p.scale_denom
    c2s = bool(p.chroma_2s) and len(im.coef) == 3 and getattr(im, "subsampling", 420) == 420
    out = []
    for ci in range(len(im.coef)):
        w, h = (g.Wd, g.Hd) if ci == 0 or c2s else (g.Wc, g.Hc)
        kk = k // 2 if (ci > 0 and c2s) else k          # reading R18: chroma at twice the scale
        v, u8 = decode_plane(im.coef[ci], qtables[im.qidx[ci]], kk, w, h, p.idct_def)
        out.append((v, u8) if with_v else u8)
    return out


def alg1_crop_window(height: int, width: int, target: int):
    vals = [ctypes.c_int32() for _ in range(4)]
    rc = lib().oracle_alg1_crop_window(height, width, target, *[ctypes.byref(v) for v in vals])
    if rc:
        raise ValueError(rc)
    return tuple(v.value for v in vals)      # (l', r', t', b')


def f64_to_f16_bits(x: float) -> int:
    return int(lib().oracle_f64_to_f16(float(x)))


# ---- baseline JPEG entropy decoding (smol_oracle_jpeg.c, T.81 F.2.2) ----
class JpegInfo(ctypes.Structure):
    _fields_ = [("width", ctypes.c_int32), ("height", ctypes.c_int32), ("ncomp", ctypes.c_int32),
                ("h", ctypes.c_int32 * 3), ("v", ctypes.c_int32 * 3), ("tq", ctypes.c_int32 * 3),
                ("blocks_w", ctypes.c_int32 * 3), ("blocks_h", ctypes.c_int32 * 3),
                ("mcus_x", ctypes.c_int32), ("mcus_y", ctypes.c_int32),
                ("restart_interval", ctypes.c_int32), ("qt", (ctypes.c_uint16 * 64) * 4)]


def jpeg_info(data: bytes) -> JpegInfo:
    info = JpegInfo()
    rc = lib().oracle_jpeg_info_of(data, len(data), ctypes.byref(info))
    if rc:
        raise ValueError(f"oracle_jpeg_info_of: {rc}")
    return info


def jpeg_decode(data: bytes):
    """-> (info, [planes [bh][bw][64] int16 natural order, absolute DC],
    qtables [4][64] uint16 natural order)."""
    info = jpeg_info(data)
    planes = [np.zeros((info.blocks_h[c], info.blocks_w[c], 64), dtype=np.int16) for c in range(info.ncomp)]
    ptrs = (ctypes.c_void_p * 3)(*([_ptr(p) for p in planes] + [None] * (3 - info.ncomp)))
    rc = lib().oracle_jpeg_decode(data, len(data), ptrs)
    if rc:
        raise ValueError(f"oracle_jpeg_decode: {rc}")
    qt = np.array([[info.qt[t][k] for k in range(64)] for t in range(4)], dtype=np.uint16)
    return info, planes, qt
