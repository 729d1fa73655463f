"""ctypes mirror of include/smol_preproc.h and the nvcc build of the library.

Argument marshalling only: every step of the path runs in the CUDA library.
There is no fallback: if the shared library is missing, loading raises.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

_PKG = os.path.dirname(os.path.abspath(__file__))
_ROOT = os.path.dirname(_PKG)
LIB_PATH = os.path.join(_PKG, "libsmol_preproc.so")
HEADER = os.path.join(_ROOT, "include", "smol_preproc.h")
_CSRC = os.path.join(_PKG, "csrc")
# translation units (compiled in parallel, then linked) and the headers they include
UNITS = ["smol_preproc.cu", "smol_inst_k1.cu", "smol_inst_k2.cu", "smol_inst_k4.cu", "smol_inst_k8.cu"]
HEADERS = ["smol_kernels.cuh", "smol_geom.cuh", "smol_compact.cuh", "smol_thumb.cuh", "smol_jpeg.cuh", "smol_launch.h"]
SOURCES = [os.path.join(_CSRC, f) for f in UNITS + HEADERS]
NVCC_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
              "-Xcompiler", "-fPIC", "-Xptxas", "-v", "-Xfatbin", "-compress-all"]

# smol_status
SMOL_OK, SMOL_ERR_INVALID, SMOL_ERR_UNSUPPORTED, SMOL_ERR_CUDA, SMOL_ERR_NOMEM, SMOL_ERR_CAPACITY = range(6)
STATUS_NAMES = {0: "OK", 1: "INVALID", 2: "UNSUPPORTED", 3: "CUDA", 4: "NOMEM", 5: "CAPACITY"}
SMOL_OUT_F32_NCHW, SMOL_OUT_F16_NCHW = 0, 1
SMOL_RESIZE_SHORT_SIDE, SMOL_RESIZE_EXACT = 0, 1
SMOL_LAYOUT_DENSE64, SMOL_LAYOUT_PACKED = 0, 1
SMOL_IDCT_BOX_MEAN, SMOL_IDCT_TRUNCATED = 0, 1

# every symbol include/smol_preproc.h declares (checked by tests/test_abi.py)
EXPORTS = ["smol_preproc_plan", "smol_preproc_run", "smol_preproc_run_host", "smol_preproc_destroy",
           "smol_preproc_output_shape", "smol_preproc_launches_per_run", "smol_debug_geometry",
           "smol_debug_run", "smol_last_error", "smol_abi_version", "smol_compact_encode",
           "smol_preproc_run_compact", "smol_jpeg_parse_header", "smol_preproc_run_jpeg",
           "smol_jpeg_decode_planes"]


class Params(ctypes.Structure):
    _fields_ = [("scale_denom", ctypes.c_int32), ("resize_mode", ctypes.c_int32),
                ("resize_short", ctypes.c_int32), ("resize_w", ctypes.c_int32),
                ("resize_h", ctypes.c_int32), ("crop_w", ctypes.c_int32), ("crop_h", ctypes.c_int32),
                ("mean", ctypes.c_float * 3), ("std", ctypes.c_float * 3),
                ("out_dtype", ctypes.c_int32), ("layout", ctypes.c_int32),
                ("tile_rows", ctypes.c_int32), ("idct_def", ctypes.c_int32),
                ("max_width", ctypes.c_int32), ("max_height", ctypes.c_int32),
                ("chroma_2s", ctypes.c_int32)]


class ImageDesc(ctypes.Structure):
    _fields_ = [("width", ctypes.c_int32), ("height", ctypes.c_int32),
                ("subsampling", ctypes.c_int32), ("qtable", ctypes.c_int32 * 3),
                ("coef", ctypes.c_void_p * 3), ("blocks_w", ctypes.c_int32 * 3),
                ("blocks_h", ctypes.c_int32 * 3), ("row_stride_bytes", ctypes.c_int32 * 3),
                ("roi_left", ctypes.c_int32), ("roi_top", ctypes.c_int32),
                ("roi_x", ctypes.c_int32), ("roi_y", ctypes.c_int32),
                ("roi_w", ctypes.c_int32), ("roi_h", ctypes.c_int32)]


class CompactImage(ctypes.Structure):
    _fields_ = [("width", ctypes.c_int32), ("height", ctypes.c_int32),
                ("subsampling", ctypes.c_int32), ("qtable", ctypes.c_int32 * 3),
                ("roi_left", ctypes.c_int32), ("roi_top", ctypes.c_int32),
                ("roi_x", ctypes.c_int32), ("roi_y", ctypes.c_int32),
                ("roi_w", ctypes.c_int32), ("roi_h", ctypes.c_int32),
                ("offset", ctypes.c_int64)]


class CompactBatchDesc(ctypes.Structure):
    _fields_ = [("n_images", ctypes.c_int32), ("images", ctypes.POINTER(CompactImage)),
                ("arena", ctypes.c_void_p), ("arena_bytes", ctypes.c_int64),
                ("qtables", ctypes.c_void_p), ("n_qtables", ctypes.c_int32)]


class JpegImage(ctypes.Structure):
    _fields_ = [("offset", ctypes.c_int64), ("size", ctypes.c_int64),
                ("roi_left", ctypes.c_int32), ("roi_top", ctypes.c_int32),
                ("roi_x", ctypes.c_int32), ("roi_y", ctypes.c_int32),
                ("roi_w", ctypes.c_int32), ("roi_h", ctypes.c_int32)]


class JpegBatchDesc(ctypes.Structure):
    _fields_ = [("n_images", ctypes.c_int32), ("images", ctypes.POINTER(JpegImage)),
                ("arena", ctypes.c_void_p), ("arena_bytes", ctypes.c_int64)]


class JpegHeader(ctypes.Structure):
    _fields_ = [("width", ctypes.c_int32), ("height", ctypes.c_int32), ("subsampling", ctypes.c_int32),
                ("ncomp", ctypes.c_int32), ("blocks_w", ctypes.c_int32 * 3), ("blocks_h", ctypes.c_int32 * 3),
                ("mcus_x", ctypes.c_int32), ("mcus_y", ctypes.c_int32), ("restart_interval", ctypes.c_int32),
                ("n_segments", ctypes.c_int32), ("scan_offset", ctypes.c_int32)]


class BatchDesc(ctypes.Structure):
    _fields_ = [("n_images", ctypes.c_int32), ("images", ctypes.POINTER(ImageDesc)),
                ("qtables", ctypes.c_void_p), ("n_qtables", ctypes.c_int32)]


class Geometry(ctypes.Structure):
    _fields_ = ([(n, ctypes.c_int32) for n in ("Wd", "Hd", "Wc", "Hc", "Wr", "Hr", "left", "top",
                                               "OW", "OH", "lx0", "lx1", "ly0", "ly1",
                                               "cx0", "cx1", "cy0", "cy1")] +
                [(n, ctypes.c_int32 * 3) for n in ("bx0", "bx1", "by0", "by1")] +
                [("roi_blocks", ctypes.c_int64), ("roi_coef_bytes", ctypes.c_int64)] +
                [(n, ctypes.c_int32) for n in ("sx0", "sy0", "sw", "sh")] +
                [("storage_coef_bytes", ctypes.c_int64)])

    def as_dict(self):
        d = {}
        for n, _ in self._fields_:
            v = getattr(self, n)
            d[n] = list(v) if isinstance(v, ctypes.Array) else v
        return d


def _stale() -> bool:
    if not os.path.exists(LIB_PATH):
        return True
    t = os.path.getmtime(LIB_PATH)
    return any(os.path.getmtime(s) > t for s in SOURCES + [HEADER])


def build(force: bool = False, verbose: bool = False, out: str = None, defines=()) -> str:
    """nvcc -gencode arch=compute_100a,code=sm_100a ... -> libsmol_preproc.so
    (in-tree): every unit compiled to an object in parallel, then linked.
    out/defines: an experiment variant (-D flags) built to another path."""
    target = out or LIB_PATH
    if out is None and not force and not _stale():
        return LIB_PATH
    from concurrent.futures import ThreadPoolExecutor
    objdir = os.path.join(_PKG, "build")
    os.makedirs(objdir, exist_ok=True)
    inc = ["-I", os.path.join(_ROOT, "include"), "-I", _CSRC]

    def compile_unit(u):
        obj = os.path.join(objdir, u.replace(".cu", f".{os.getpid()}.{abs(hash(target))}.o"))
        cmd = ["nvcc", *NVCC_FLAGS, *[f"-D{d}" for d in defines], *inc, "-c", "-o", obj, os.path.join(_CSRC, u)]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed ({' '.join(cmd)}):\n{r.stderr}")
        return obj, r.stderr

    with ThreadPoolExecutor(len(UNITS)) as ex:
        res = list(ex.map(compile_unit, UNITS))
    tmp = target + f".tmp{os.getpid()}"
    cmd = ["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", tmp] + [o for o, _ in res]
    r = subprocess.run(cmd, capture_output=True, text=True)
    for o, _ in res:
        os.remove(o)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc link failed ({' '.join(cmd)}):\n{r.stderr}")
    if verbose:
        print("".join(e for _, e in res))
    os.replace(tmp, target)
    return target


_lib = None


def lib():
    """Load the CUDA library; raises if it was not built (no CPU fallback)."""
    global _lib
    if _lib is None:
        path = os.environ.get("SMOL_LIB", LIB_PATH)      # experiment override (same ABI)
        if not os.path.exists(path):
            raise RuntimeError(f"{path} missing: run __graft_entry__.build() "
                               "(the Smol path has no CPU fallback)")
        L = ctypes.CDLL(path)
        P = ctypes.POINTER
        vp = ctypes.c_void_p
        L.smol_preproc_plan.argtypes = [P(Params), ctypes.c_int32, P(vp)]
        L.smol_preproc_run.argtypes = [vp, P(BatchDesc), vp, vp]
        L.smol_preproc_run_host.argtypes = [vp, P(BatchDesc), vp, vp]
        L.smol_preproc_destroy.argtypes = [vp]
        L.smol_preproc_destroy.restype = None
        L.smol_preproc_output_shape.argtypes = [vp] + [P(ctypes.c_int32)] * 3
        L.smol_preproc_launches_per_run.argtypes = [vp]
        L.smol_debug_geometry.argtypes = [P(Params), P(ImageDesc), P(Geometry)]
        L.smol_debug_run.argtypes = [vp, P(BatchDesc), vp, vp, vp, vp, vp,
                                     ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, vp]
        L.smol_last_error.argtypes = []
        L.smol_last_error.restype = ctypes.c_char_p
        L.smol_abi_version.argtypes = []
        L.smol_compact_encode.argtypes = [P(Params), P(ImageDesc), vp, ctypes.c_int64, P(ctypes.c_int64)]
        L.smol_preproc_run_compact.argtypes = [vp, P(CompactBatchDesc), vp, vp]
        L.smol_jpeg_parse_header.argtypes = [ctypes.c_char_p, ctypes.c_int64, P(JpegHeader)]
        L.smol_preproc_run_jpeg.argtypes = [vp, P(JpegBatchDesc), vp, vp]
        L.smol_jpeg_decode_planes.argtypes = [P(JpegBatchDesc), ctypes.POINTER(vp), vp]
        for name in EXPORTS:
            f = getattr(L, name)
            if f.restype is ctypes.c_int:           # ctypes default
                f.restype = ctypes.c_int32
        _lib = L
    return _lib


class SmolError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"smol status {STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status


def check(status: int) -> None:
    if status != SMOL_OK:
        raise SmolError(status, lib().smol_last_error().decode())
