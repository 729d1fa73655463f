"""Packed-for-scale coefficient layout (include/smol_preproc.h PACKED).

The kept index sets are pinned against the method itself: a coefficient that
the packed layout drops must not influence the decoded samples at that scale
(the oracle decodes it to exactly 0, and scipy's box mean to ~0); every kept
coefficient must influence them."""
import numpy as np
import pytest
from scipy import fft

from paper_2007_13005_b200 import layout
import paper_2007_13005_b200 as smol


@pytest.mark.parametrize("k", [2, 4, 8])
def test_dropped_coefficients_do_not_contribute(oracle_mod, k):
    keep = set(layout.index_set(k))
    q = np.ones(64, np.uint16)
    P = 8 // k
    for idx in range(64):
        c = np.zeros((1, 1, 64), np.int16)
        c[0, 0, idx] = 100
        v, _ = oracle_mod.decode_plane(c, q, k, P, P)
        ref = fft.idctn(c[0, 0].reshape(8, 8).astype(np.float64), norm="ortho").reshape(P, k, P, k).mean(axis=(1, 3))
        if idx in keep:
            assert np.abs(ref).max() > 1e-3, (k, idx)
        else:
            assert np.all(v == 0.0) and np.abs(ref).max() < 1e-9, (k, idx)


@pytest.mark.parametrize("k,e", [(1, 64), (2, 52), (4, 28), (8, 1)])
def test_pack_plane_shapes_and_content(k, e):
    rng = np.random.default_rng(k)
    c = rng.integers(-500, 500, size=(3, 5, 64)).astype(np.int16)
    p = layout.pack_plane(c, k)
    assert p.shape[0] == 3 and (p.shape[1] * 2) % 16 == 0 and p.shape[1] >= 5 * e
    idx = layout.index_set(k)
    blocks = p[:, :5 * e].reshape(3, 5, e)
    assert np.array_equal(blocks[:, :, :len(idx)], c[:, :, idx])
    assert np.all(blocks[:, :, len(idx):] == 0)


def test_geometry_bytes_per_layout():
    # algorithmic bytes: K_s used coefficients per ROI block,
    # independent of the layout; storage bytes: what each layout holds
    for k, ks, dense, packed in ((1, 64, 128, 128), (2, 49, 128, 104), (4, 25, 128, 56), (8, 1, 32, 2)):
        gd = smol.geometry(smol.make_params(scale_denom=k, resize_mode="exact", resize_w=64, resize_h=64), 500, 375)
        gp = smol.geometry(smol.make_params(scale_denom=k, resize_mode="exact", resize_w=64, resize_h=64,
                                            layout="packed"), 500, 375)
        assert gd["roi_coef_bytes"] == gp["roi_coef_bytes"] == gd["roi_blocks"] * 2 * ks
        assert ks == len(layout.index_set(k))
        assert gd["storage_coef_bytes"] == gd["roi_blocks"] * dense
        assert gp["storage_coef_bytes"] == gp["roi_blocks"] * packed


def test_survey_8d_bytes_per_image():
    """packed ROI coefficient bytes per image."""
    import synth
    want = {"c2": 344064, "c3a": 271852, "c3b": 138700, "c4": 1366, "c5": 2436000}
    for name, b in want.items():
        cfg = synth.CONFIGS[name]
        g = smol.geometry(smol.params_from_config(cfg, layout="packed"), cfg.width, cfg.height)
        assert g["roi_coef_bytes"] == b, (name, g["roi_coef_bytes"])
