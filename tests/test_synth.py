"""The seeded generator: deterministic, right shapes, valid ranges."""
import numpy as np

import synth


def test_deterministic_and_shapes():
    cfg = synth.CONFIGS["c1"]
    a, qa = synth.distinct_images(cfg, n_distinct=3)
    b, qb = synth.distinct_images(cfg, n_distinct=3)
    assert np.array_equal(qa, qb)
    for x, y in zip(a, b):
        for ci in range(3):
            assert np.array_equal(x.coef[ci], y.coef[ci])
    im = a[0]
    assert im.blocks_w == [8, 4, 4] and im.blocks_h == [8, 4, 4]
    assert all(c.dtype == np.int16 for c in im.coef)


def test_mcu_padding_odd_sizes():
    qt = synth.quant_tables(75)
    rng = np.random.default_rng(0)
    im = synth.make_image(rng, 17, 33, qt)
    assert im.blocks_w == [4, 2, 2] and im.blocks_h == [6, 3, 3]


def test_quant_tables_ijg():
    q50 = synth.quant_tables(50)
    assert np.array_equal(q50[0], synth.ANNEX_K1)        # scale 100 at q=50
    q95 = synth.quant_tables(95)
    assert q95[0][0] == 2 and q95.min() >= 1


def test_stress_range():
    qt = synth.quant_tables(75)
    im = synth.stress_image(np.random.default_rng(1), 64, 48, qt)
    for ci in range(3):
        D = im.coef[ci].astype(np.int64) * qt[0 if ci == 0 else 1].astype(np.int64)
        assert np.abs(D).max() <= 2047
