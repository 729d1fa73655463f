"""CPU-side checks of the C-ABI library: it loads, exports every symbol the
header declares, and its host-only geometry (smol_debug_geometry) agrees with
the oracle's independent geometry and with an exact-rational footprint
computation.  No compute calls (no GPU here)."""
import ctypes
import os
import re
from fractions import Fraction

import numpy as np
import pytest

import paper_2007_13005_b200 as smol
from paper_2007_13005_b200 import _native

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def native():
    _native.build()
    return _native.lib()


def test_exports_every_declared_symbol(native):
    hdr = open(os.path.join(ROOT, "include", "smol_preproc.h")).read()
    declared = set(re.findall(r"^\s*(?:int32_t|void|const char\*)\s+(smol_\w+)\s*\(", hdr, re.M))
    assert declared == set(_native.EXPORTS)
    for name in declared:
        assert hasattr(native, name), name
    assert native.smol_abi_version() == 3


def test_library_is_sm100a(native):
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", _native.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def _src_tap(d, n_in, n_out):
    """R8 in exact rationals: src = max(0, (d+1/2) in/out - 1/2)."""
    src = max(Fraction(0), (Fraction(2 * d + 1, 2) * n_in) / n_out - Fraction(1, 2))
    i0 = int(src)
    return i0, min(i0 + 1, n_in - 1)


@pytest.mark.parametrize("k", [1, 2, 4, 8])
def test_geometry_matches_oracle_and_rationals(native, oracle_mod, k):
    rng = np.random.default_rng(31 + k)
    sizes = [(500, 375), (375, 500), (161, 161), (1920, 1080), (64, 64), (97, 61), (33, 17)]
    sizes += [(int(a), int(b)) for a, b in rng.integers(16, 900, size=(25, 2))]
    for (w, h) in sizes:
        for mode in ("short", "exact"):
            if mode == "short":
                kw = dict(resize_short=max(8, 256 // k), crop_w=max(4, 224 // k), crop_h=max(4, 200 // k))
            else:
                kw = dict(resize_w=64, resize_h=48)
            p = smol.make_params(scale_denom=k, resize_mode=mode, **kw)
            po = oracle_mod.make_params(scale_denom=k, resize_mode=mode, **kw)
            try:
                og = oracle_mod.geometry(po, w, h).as_dict()
            except ValueError:
                with pytest.raises(smol.SmolError):
                    smol.geometry(p, w, h)
                continue
            g = smol.geometry(p, w, h)
            for key in ("Wd", "Hd", "Wc", "Hc", "Wr", "Hr", "left", "top", "OW", "OH"):
                assert g[key] == og[key], (w, h, k, mode, key)
            lx0 = _src_tap(g["left"], g["Wd"], g["Wr"])[0]
            lx1 = _src_tap(g["left"] + g["OW"] - 1, g["Wd"], g["Wr"])[1]
            ly0 = _src_tap(g["top"], g["Hd"], g["Hr"])[0]
            ly1 = _src_tap(g["top"] + g["OH"] - 1, g["Hd"], g["Hr"])[1]
            assert (g["lx0"], g["lx1"], g["ly0"], g["ly1"]) == (lx0, lx1, ly0, ly1)
            P = 8 // k
            # luma columns are decoded in groups of 4 (2x2 quads, widened to
            # 4-alignment, within the image's valid block columns)
            assert (g["bx0"][0], g["bx1"][0]) == ((lx0 & ~3) // P, min((lx1 | 3) // P, -(-w // 8) - 1))
            cx0, cx1 = max(0, (lx0 - 1) // 2), min(g["Wc"] - 1, (lx1 + 1) // 2)
            assert (g["bx0"][1], g["bx1"][1]) == (cx0 // P, cx1 // P)


def test_c2_roi_block_count(native):
    # SURVEY §8(a) row a1 [derived]: c2 taps x 85..413, y 23..351; ROI 1764 Y +
    # 924 C = 2688 of 4608 blocks.
    p = smol.make_params(scale_denom=1, resize_short=256, crop_w=224, crop_h=224)
    g = smol.geometry(p, 500, 375)
    assert (g["lx0"], g["lx1"], g["ly0"], g["ly1"]) == (85, 413, 23, 351)
    assert g["roi_blocks"] == 2688
    assert g["roi_coef_bytes"] == 2688 * 128


@pytest.mark.parametrize("bad,msg", [
    (dict(scale_denom=3), "scale_denom"),
    (dict(std=(0.2, 0.0, 0.2)), "std"),
    (dict(resize_mode="short", crop_w=0, crop_h=0), "crop"),
    (dict(resize_mode="exact", resize_w=32, resize_h=32, crop_w=64, crop_h=64), "crop"),
])
def test_param_validation(native, bad, msg):
    kw = dict(scale_denom=1, resize_mode="short", resize_short=256, crop_w=224, crop_h=224)
    kw.update(bad)
    p = smol.make_params(**kw)
    with pytest.raises(smol.SmolError) as e:
        smol.geometry(p, 500, 375)
    assert e.value.status == _native.SMOL_ERR_INVALID
    assert msg in str(e.value)


def test_unsupported_subsampling_and_crop_too_big(native):
    p = smol.make_params(scale_denom=1, resize_short=256, crop_w=224, crop_h=224)
    d = smol._desc_for(500, 375, [63, 32, 32], [47, 24, 24])
    d.subsampling = 411                      # (4:1:1 is not a supported sampling)
    g = _native.Geometry()
    assert native.smol_debug_geometry(ctypes.byref(p), ctypes.byref(d), ctypes.byref(g)) == _native.SMOL_ERR_UNSUPPORTED
    # 4:2:2 / 4:4:4 chroma sizes (T.81 A.1.1) agree with the oracle
    import oracle
    po = oracle.make_params(scale_denom=2, resize_mode="exact", resize_w=64, resize_h=64)
    for ss in (420, 422, 444):
        gs = smol.geometry(smol.make_params(scale_denom=2, resize_mode="exact", resize_w=64, resize_h=64),
                           500, 375, subsampling=ss)
        go = oracle.geometry(po, 500, 375, ss)
        assert (gs["Wc"], gs["Hc"], gs["Wd"], gs["Hd"]) == (go.Wc, go.Hc, go.Wd, go.Hd)
    p2 = smol.make_params(scale_denom=8, resize_short=16, crop_w=224, crop_h=224)
    with pytest.raises(smol.SmolError):
        smol.geometry(p2, 500, 375)
