"""B200-native Smol preprocessing hot path (arXiv 2007.13005, §2 steps 1-4 and
§6.4 partial / reduced-fidelity decoding) -- thin Python binding.

The product is the C-ABI library ``libsmol_preproc.so`` (include/smol_preproc.h)
built from ``csrc/`` for sm_100a.  This module only marshals arguments:
coefficient planes live in a torch-allocated arena (device memory or pinned
host memory), descriptors are ctypes structs, and every computation runs in
the fused CUDA kernel.  There is no CPU fallback: without the library every
call raises.
"""
from __future__ import annotations

import ctypes
from typing import Optional, Sequence, Tuple

import numpy as np

from ._native import (BatchDesc, CompactBatchDesc, CompactImage, Geometry, ImageDesc, JpegBatchDesc,
                      JpegHeader, JpegImage, Params,
                      SmolError, build, check, lib,
                      SMOL_OUT_F16_NCHW, SMOL_OUT_F32_NCHW, SMOL_RESIZE_EXACT,
                      SMOL_RESIZE_SHORT_SIDE, SMOL_LAYOUT_DENSE64, SMOL_LAYOUT_PACKED, EXPORTS,
                      SMOL_IDCT_BOX_MEAN, SMOL_IDCT_TRUNCATED,
                      LIB_PATH)
from .layout import block_elems, pack_plane

__all__ = ["make_params", "params_from_config", "geometry", "CoefBatch", "CompactBatch", "JpegBatch",
           "jpeg_header",
           "compact_encode", "Plan", "SmolError",
           "build", "lib", "EXPORTS", "LIB_PATH"]

IMAGENET_MEAN = (0.485, 0.456, 0.406)
IMAGENET_STD = (0.229, 0.224, 0.225)


def make_params(scale_denom: int = 1, resize_mode: str = "short", resize_short: int = 256,
                resize_w: int = 0, resize_h: int = 0, crop_w: int = 0, crop_h: int = 0,
                mean=IMAGENET_MEAN, std=IMAGENET_STD, out_dtype: str = "f32",
                tile_rows: int = 0, layout: str = "dense", idct_def: str = "box",
                max_size: Optional[Tuple[int, int]] = None, chroma_2s: bool = False) -> Params:
    p = Params()
    p.scale_denom = scale_denom
    p.resize_mode = SMOL_RESIZE_SHORT_SIDE if resize_mode == "short" else SMOL_RESIZE_EXACT
    p.resize_short, p.resize_w, p.resize_h = resize_short, resize_w, resize_h
    p.crop_w, p.crop_h = crop_w, crop_h
    p.mean = (ctypes.c_float * 3)(*mean)
    p.std = (ctypes.c_float * 3)(*std)
    p.out_dtype = SMOL_OUT_F16_NCHW if out_dtype == "f16" else SMOL_OUT_F32_NCHW
    p.layout = SMOL_LAYOUT_PACKED if layout == "packed" else SMOL_LAYOUT_DENSE64
    p.tile_rows = tile_rows
    p.idct_def = SMOL_IDCT_TRUNCATED if idct_def == "truncated" else SMOL_IDCT_BOX_MEAN
    p.max_width, p.max_height = max_size if max_size is not None else (0, 0)
    p.chroma_2s = 1 if chroma_2s else 0
    return p


def batch_for(params: Params, images, qtables, **kw) -> "CoefBatch":
    """CoefBatch in the layout the plan's params expect."""
    return CoefBatch(images, qtables, layout="packed" if params.layout == SMOL_LAYOUT_PACKED else "dense",
                     scale_denom=params.scale_denom, truncated=params.idct_def == SMOL_IDCT_TRUNCATED, **kw)


def params_from_config(cfg, **kw) -> Params:
    """Params for a synth.Config (BASELINE.json workload)."""
    args = dict(scale_denom=cfg.scale_denom, resize_mode=cfg.resize_mode,
                resize_short=cfg.resize_short, resize_w=cfg.resize_w, resize_h=cfg.resize_h,
                crop_w=cfg.crop_w, crop_h=cfg.crop_h, out_dtype=cfg.out_dtype)
    args.update(kw)
    return make_params(**args)


def _desc_for(width, height, blocks_w, blocks_h, qidx=(0, 1, 1), roi=None, strides=None,
              subsampling=None, roi_rect=None) -> ImageDesc:
    """Descriptor of a 3-plane image (4:2:0 unless `subsampling` says 422 /
    444) or a grayscale one (1 plane: subsampling 400, chroma fields zero).
    roi: crop-window origin (left, top) in resized coordinates; roi_rect:
    (x, y, w, h) ROI rectangle in SOF pixels."""
    d = ImageDesc()
    gray = len(blocks_w) == 1
    d.width, d.height = width, height
    d.subsampling = 400 if gray else (subsampling or 420)
    if roi_rect is not None:
        d.roi_x, d.roi_y, d.roi_w, d.roi_h = roi_rect
    d.qtable = (ctypes.c_int32 * 3)(*(tuple(qidx) + (0, 0, 0))[:3])
    for c in range(len(blocks_w)):
        d.blocks_w[c], d.blocks_h[c] = blocks_w[c], blocks_h[c]
        d.row_stride_bytes[c] = blocks_w[c] * 128 if strides is None else strides[c]
    d.roi_left, d.roi_top = roi if roi is not None else (-1, -1)
    return d


SUBSAMPLING = {420: (2, 2), 422: (2, 1), 444: (1, 1)}


def geometry(params: Params, width: int, height: int, roi=None, gray: bool = False,
             subsampling: int = 420, roi_rect=None) -> dict:
    """Host-only geometry of one image (smol_debug_geometry)."""
    n = 1 if gray else 3
    hs, vs = SUBSAMPLING.get(subsampling, (2, 2))
    bw = [(width + 7) // 8] + [-(-width // (8 * hs))] * 2
    bh = [(height + 7) // 8] + [-(-height // (8 * vs))] * 2
    d = _desc_for(width, height, bw[:n], bh[:n], roi=roi, subsampling=subsampling, roi_rect=roi_rect)
    g = Geometry()
    check(lib().smol_debug_geometry(ctypes.byref(params), ctypes.byref(d), ctypes.byref(g)))
    return g.as_dict()


class CoefBatch:
    """Entropy-decoded coefficient planes of N images in one torch arena.

    images: sequence of objects with .width, .height, .coef (3 int16 arrays
    [bh][bw][64]) and .qidx; qtables: [nq][64] uint16.  location: "device"
    (HBM, for smol_preproc_run) or "pinned" (page-locked host memory, for the
    end-to-end smol_preproc_run_host path).  layout/scale_denom select the
    plan's coefficient layout: "packed" keeps only the coefficients the scale
    uses (layout.pack_plane; what a host entropy decoder would emit).
    """

    def __init__(self, images: Sequence, qtables: np.ndarray, location: str = "device",
                 device: Optional[int] = None, rois: Optional[Sequence] = None,
                 layout: str = "dense", scale_denom: int = 1, roi_rects: Optional[Sequence] = None,
                 truncated: bool = False):
        import torch
        self.n = len(images)
        k = scale_denom if layout == "packed" else 1
        planes = []
        cache = {}
        for im in images:
            key = id(im)
            if key not in cache:
                cache[key] = [pack_plane(np.ascontiguousarray(c, dtype=np.int16), k, truncated) for c in im.coef]
            planes.append(cache[key])
        sizes = [[int(p.size) for p in ps] for ps in planes]
        total = int(sum(sum(s) for s in sizes))
        host = np.empty(max(total, 8), np.int16)
        offs = []
        o = 0
        for ps, s in zip(planes, sizes):
            oo = []
            for ci in range(len(ps)):
                host[o:o + s[ci]] = ps[ci].ravel()
                oo.append(o)
                o += s[ci]                      # every plane row is a multiple of 16 bytes
            offs.append(oo)
        qt = np.ascontiguousarray(qtables, dtype=np.uint16).view(np.int16)
        dev = torch.device("cuda", torch.cuda.current_device() if device is None else device)
        if location == "device":
            self.arena = torch.from_numpy(host).to(dev)
            self.qtables = torch.from_numpy(qt.copy()).to(dev)
        elif location == "pinned":
            self.arena = torch.from_numpy(host).pin_memory()
            self.qtables = torch.from_numpy(qt.copy()).to(dev)
        else:
            raise ValueError(location)
        self.location = location
        self.coef_bytes = int(self.arena.numel()) * 2
        base = self.arena.data_ptr()
        self.descs = (ImageDesc * max(self.n, 1))()
        for i, (im, oo) in enumerate(zip(images, offs)):
            roi = rois[i] if rois is not None else None
            d = _desc_for(im.width, im.height, [c.shape[1] for c in im.coef],
                          [c.shape[0] for c in im.coef], tuple(im.qidx), roi,
                          strides=[2 * p.shape[1] for p in planes[i]],
                          subsampling=getattr(im, "subsampling", 420),
                          roi_rect=None if roi_rects is None else roi_rects[i])
            for ci in range(len(im.coef)):
                d.coef[ci] = base + 2 * oo[ci]
            self.descs[i] = d
        self.desc = BatchDesc()
        self.desc.n_images = self.n
        self.desc.images = ctypes.cast(self.descs, ctypes.POINTER(ImageDesc))
        self.desc.qtables = self.qtables.data_ptr()
        self.desc.n_qtables = int(qtables.shape[0])


def compact_encode(params: Params, im, roi=None, roi_rect=None) -> np.ndarray:
    """One image's compact record (smol_compact_encode, host only) as uint8.

    im: object with .width, .height, .coef (3 int16 [bh][bw][64]) and .qidx;
    the planes are first put in the params' layout (what the host entropy
    decoder holds), then the C encoder keeps the ROI blocks' nonzero used
    coefficients (include/smol_preproc.h "Compact coefficient transport")."""
    k = params.scale_denom if params.layout == SMOL_LAYOUT_PACKED else 1
    planes = [pack_plane(np.ascontiguousarray(c, dtype=np.int16), k, params.idct_def == SMOL_IDCT_TRUNCATED)
              for c in im.coef]
    d = _desc_for(im.width, im.height, [c.shape[1] for c in im.coef], [c.shape[0] for c in im.coef],
                  tuple(im.qidx), roi, strides=[2 * p.shape[1] for p in planes],
                  subsampling=getattr(im, "subsampling", 420), roi_rect=roi_rect)
    for ci in range(len(planes)):
        d.coef[ci] = planes[ci].ctypes.data
    n = ctypes.c_int64()
    check(lib().smol_compact_encode(ctypes.byref(params), ctypes.byref(d), None, 0, ctypes.byref(n)))
    rec = np.zeros(n.value, np.uint8)
    check(lib().smol_compact_encode(ctypes.byref(params), ctypes.byref(d), rec.ctypes.data, n.value,
                                    ctypes.byref(n)))
    return rec


class CompactBatch:
    """N images as compact records (the end-to-end transport, SURVEY §8(f)
    N1) in one arena: location "pinned" (page-locked host memory, copied by
    smol_preproc_run_compact in one DMA) or "device".  Records are encoded
    for `params` (layout, scale and crop fix the ROI and element set)."""

    def __init__(self, params: Params, images: Sequence, qtables: np.ndarray, location: str = "pinned",
                 device: Optional[int] = None, rois: Optional[Sequence] = None,
                 roi_rects: Optional[Sequence] = None):
        import torch
        self.n = len(images)
        cache = {}
        recs = []
        for i, im in enumerate(images):
            roi = rois[i] if rois is not None else None
            rr = roi_rects[i] if roi_rects is not None else None
            key = (id(im), roi, rr)
            if key not in cache:
                cache[key] = compact_encode(params, im, roi, rr)
            recs.append(cache[key])
        offs, o = [], 0
        for r in recs:
            offs.append(o)
            o += r.size                           # records are multiples of 16 bytes
        host = np.zeros(max(o, 16), np.uint8)
        for r, oo in zip(recs, offs):
            host[oo:oo + r.size] = r
        qt = np.ascontiguousarray(qtables, dtype=np.uint16).view(np.int16)
        dev = torch.device("cuda", torch.cuda.current_device() if device is None else device)
        if location == "pinned":
            self.arena = torch.from_numpy(host).pin_memory()
        elif location == "device":
            self.arena = torch.from_numpy(host).to(dev)
        else:
            raise ValueError(location)
        self.location = location
        self.qtables = torch.from_numpy(qt.copy()).to(dev)
        self.arena_bytes = int(o)
        self.images = (CompactImage * max(self.n, 1))()
        for i, (im, oo) in enumerate(zip(images, offs)):
            ci = CompactImage()
            ci.width, ci.height = im.width, im.height
            ci.subsampling = 400 if len(im.coef) == 1 else getattr(im, "subsampling", 420)
            ci.qtable = (ctypes.c_int32 * 3)(*(tuple(im.qidx) + (0, 0, 0))[:3])
            roi = rois[i] if rois is not None else None
            ci.roi_left, ci.roi_top = roi if roi is not None else (-1, -1)
            if roi_rects is not None and roi_rects[i] is not None:
                ci.roi_x, ci.roi_y, ci.roi_w, ci.roi_h = roi_rects[i]
            ci.offset = oo
            self.images[i] = ci
        self.desc = CompactBatchDesc()
        self.desc.n_images = self.n
        self.desc.images = ctypes.cast(self.images, ctypes.POINTER(CompactImage))
        self.desc.arena = self.arena.data_ptr()
        self.desc.arena_bytes = max(self.arena_bytes, 16)
        self.desc.qtables = self.qtables.data_ptr()
        self.desc.n_qtables = int(qtables.shape[0])


def jpeg_header(data: bytes) -> dict:
    """smol_jpeg_parse_header: the library's reading of a JPEG file's header."""
    h = JpegHeader()
    check(lib().smol_jpeg_parse_header(bytes(data), len(data), ctypes.byref(h)))
    return {"width": h.width, "height": h.height, "subsampling": h.subsampling, "ncomp": h.ncomp,
            "blocks_w": list(h.blocks_w)[:h.ncomp], "blocks_h": list(h.blocks_h)[:h.ncomp],
            "mcus_x": h.mcus_x, "mcus_y": h.mcus_y, "restart_interval": h.restart_interval,
            "n_segments": h.n_segments, "scan_offset": h.scan_offset}


class JpegBatch:
    """N JPEG files in one pinned host arena, for
    smol_preproc_run_jpeg (headers parsed on the host, entropy decoding on the
    GPU).  rois / roi_rects as for CompactBatch."""

    def __init__(self, files: Sequence[bytes], rois: Optional[Sequence] = None,
                 roi_rects: Optional[Sequence] = None):
        import torch
        self.n = len(files)
        offs, o, seen = [], 0, {}
        for f in files:                 # identical file objects share one copy
            k = id(f)
            if k not in seen:
                seen[k] = o
                o += (len(f) + 15) & ~15
            offs.append(seen[k])
        host = np.zeros(max(o, 16), np.uint8)
        for f, oo in zip(files, offs):
            host[oo:oo + len(f)] = np.frombuffer(f, np.uint8)
        self.arena = torch.from_numpy(host).pin_memory()
        self.arena_bytes = int(max(o, 16))
        self.file_bytes = int(sum(len(f) for f in files))
        self.images = (JpegImage * max(self.n, 1))()
        for i, (f, oo) in enumerate(zip(files, offs)):
            ji = JpegImage()
            ji.offset, ji.size = oo, len(f)
            roi = rois[i] if rois is not None else None
            ji.roi_left, ji.roi_top = roi if roi is not None else (-1, -1)
            if roi_rects is not None and roi_rects[i] is not None:
                ji.roi_x, ji.roi_y, ji.roi_w, ji.roi_h = roi_rects[i]
            self.images[i] = ji
        self.desc = JpegBatchDesc()
        self.desc.n_images = self.n
        self.desc.images = ctypes.cast(self.images, ctypes.POINTER(JpegImage))
        self.desc.arena = self.arena.data_ptr()
        self.desc.arena_bytes = self.arena_bytes

    def decode_planes(self, stream=None):
        """smol_jpeg_decode_planes: every block of every file, Huffman-decoded
        on the GPU -> per image a list of int16 device planes [bh][bw][64]."""
        import torch
        out, ptrs = [], []
        for i in range(self.n):
            f = bytes(self.arena[self.images[i].offset:self.images[i].offset + self.images[i].size].numpy())
            h = jpeg_header(f)
            pl = [torch.zeros((h["blocks_h"][c], h["blocks_w"][c], 64), dtype=torch.int16, device="cuda")
                  for c in range(h["ncomp"])]
            out.append(pl)
            ptrs += [p.data_ptr() for p in pl] + [None] * (3 - len(pl))
        arr = (ctypes.c_void_p * max(len(ptrs), 1))(*ptrs)
        s = torch.cuda.current_stream() if stream is None else stream
        check(lib().smol_jpeg_decode_planes(ctypes.byref(self.desc), arr, s.cuda_stream))
        return out


class Plan:
    """smol_preproc_plan on the current CUDA device."""

    def __init__(self, params: Params, max_images: int):
        self.params = params
        self._h = ctypes.c_void_p()
        check(lib().smol_preproc_plan(ctypes.byref(params), int(max_images), ctypes.byref(self._h)))
        c, h, w = ctypes.c_int32(), ctypes.c_int32(), ctypes.c_int32()
        check(lib().smol_preproc_output_shape(self._h, ctypes.byref(c), ctypes.byref(h), ctypes.byref(w)))
        self.out_shape = (c.value, h.value, w.value)
        self.max_images = max_images

    @property
    def out_dtype(self):
        import torch
        return torch.float16 if self.params.out_dtype == SMOL_OUT_F16_NCHW else torch.float32

    def launches_per_run(self) -> int:
        return int(lib().smol_preproc_launches_per_run(self._h))

    def new_output(self, n: int):
        import torch
        return torch.empty((n,) + self.out_shape, dtype=self.out_dtype, device="cuda")

    @staticmethod
    def _stream(stream) -> int:
        import torch
        s = torch.cuda.current_stream() if stream is None else stream
        return s.cuda_stream

    def run(self, batch, out=None, stream=None):
        if out is None:
            out = self.new_output(batch.n)
        if isinstance(batch, CompactBatch):
            check(lib().smol_preproc_run_compact(self._h, ctypes.byref(batch.desc), out.data_ptr(),
                                                 self._stream(stream)))
            return out
        if isinstance(batch, JpegBatch):
            check(lib().smol_preproc_run_jpeg(self._h, ctypes.byref(batch.desc), out.data_ptr(),
                                              self._stream(stream)))
            return out
        fn = lib().smol_preproc_run_host if batch.location == "pinned" else lib().smol_preproc_run
        check(fn(self._h, ctypes.byref(batch.desc), out.data_ptr(), self._stream(stream)))
        return out

    def debug_run(self, batch: CoefBatch, geoms: Sequence[dict], out=None, stream=None):
        """Fused kernel with its debug store: returns (out, Y, Cb, Cr, RGB) with
        int16 planes (-1 where the kernel did not write)."""
        import torch
        if out is None:
            out = self.new_output(batch.n)
        g = geoms
        sy = max(d["Wd"] * d["Hd"] for d in g)
        sc = max(d["Wc"] * d["Hc"] for d in g)
        y = torch.full((batch.n, sy), -1, dtype=torch.int16, device="cuda")
        cb = torch.full((batch.n, sc), -1, dtype=torch.int16, device="cuda")
        cr = torch.full((batch.n, sc), -1, dtype=torch.int16, device="cuda")
        rgb = torch.full((batch.n, 3 * sy), -1, dtype=torch.int16, device="cuda")
        check(lib().smol_debug_run(self._h, ctypes.byref(batch.desc), out.data_ptr(), y.data_ptr(),
                                   cb.data_ptr(), cr.data_ptr(), rgb.data_ptr(), sy, sc, 3 * sy,
                                   self._stream(stream)))
        return out, y, cb, cr, rgb

    def close(self):
        if self._h:
            lib().smol_preproc_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
