"""Exhaustive check of the CUDA kernel's colour-conversion recipe (reading R6)
against exact rational JFIF, for every (Y, chroma) input: Y in [0, 255],
c16 in [0, 4080] (chroma in 1/16 units after the 4:2:0 triangle filter).

The kernel (smol_kernels.cuh: colour) computes R and B in fp32 as
  t = fmaf(float(c16), k, float(Y) + c),  value = clamp(floor(t), 0, 255)
with k = fl32(1.402/16) | fl32(1.772/16), c = fl32(1/2 - 2048*1.402/16) |
fl32(1/2 - 2048*1.772/16 + 2^-13) (constants from smol_preproc.cu: init_basis),
and G in unsigned 32-bit integers.  This test emulates those exact IEEE fp32
operations in numpy (fp32 add with RNE; the FMA's exact product+sum in
float64, which is exact for these magnitudes, then one RNE rounding to fp32)
and compares with exact integer arithmetic.  It pins the recipe, not the
compiled kernel; GPU parity tests pin the kernel.
"""
import numpy as np

Y = np.arange(256, dtype=np.int64)[:, None]
C = np.arange(4081, dtype=np.int64)[None, :]


def exact(num_coef):
    # floor((2e6 Y + 1e6 + a (c16 - 2048)) / 2e6), clamped
    num = 2_000_000 * Y + 1_000_000 + num_coef * (C - 2048)
    return np.clip(np.floor_divide(num, 2_000_000), 0, 255)


def emulate(k64, c64):
    k = np.float32(k64)
    c = np.float32(c64)
    t1 = (Y.astype(np.float32) + c).astype(np.float32)             # fp32 add, RNE
    exact_sum = C.astype(np.float64) * np.float64(k) + t1.astype(np.float64)
    t = exact_sum.astype(np.float32)                               # one RNE rounding
    return np.clip(np.floor(t.astype(np.float64)), 0, 255).astype(np.int64)


def test_red_fp32_recipe_exact():
    got = emulate(1.402 / 16, 0.5 - 2048 * 1.402 / 16)
    assert np.array_equal(got, exact(175250))


def test_blue_fp32_recipe_exact_including_ties():
    got = emulate(1.772 / 16, 0.5 - 2048 * 1.772 / 16 + 1 / 8192)
    exp = exact(221500)
    assert np.array_equal(got, exp)
    # the two exact ties (Cb - 128 = +-125 -> c16 = 48, 4048) round up
    for c16 in (48, 4048):
        num = 2_000_000 * Y[:, 0] + 1_000_000 + 221500 * (c16 - 2048)
        assert np.all(num % 2_000_000 == 0)


def test_fp32_margin_unclamped():
    # margin of the unclamped fp32 values to the nearest floor boundary: the
    # computed t never crosses an integer the exact value does not reach
    for (a, k64, c64) in ((175250, 1.402 / 16, 0.5 - 2048 * 1.402 / 16),
                          (221500, 1.772 / 16, 0.5 - 2048 * 1.772 / 16 + 1 / 8192)):
        k, c = np.float32(k64), np.float32(c64)
        t1 = (Y.astype(np.float32) + c).astype(np.float32)
        t = (C.astype(np.float64) * np.float64(k) + t1.astype(np.float64)).astype(np.float32)
        num = 2_000_000 * Y + 1_000_000 + a * (C - 2048)
        assert np.array_equal(np.floor(t.astype(np.float64)).astype(np.int64), np.floor_divide(num, 2_000_000))


def test_green_unsigned_integer_recipe():
    cb = np.arange(4081, dtype=np.uint64)[:, None]
    cr = np.arange(0, 4081, 7, dtype=np.uint64)[None, :]
    u = (np.uint64(543917632) - np.uint64(43017) * cb - np.uint64(89267) * cr)
    assert u.min() >= 0 and u.max() < 2 ** 32
    q = (u // np.uint64(2_000_000)).astype(np.int64)
    for y in (0, 1, 77, 128, 200, 255):
        got = np.clip(y + q - 136, 0, 255)
        num = (2_000_000 * y + 1_000_000 - 43017 * (cb.astype(np.int64) - 2048)
               - 89267 * (cr.astype(np.int64) - 2048))
        assert np.array_equal(got, np.clip(np.floor_divide(num, 2_000_000), 0, 255))
