// smol_thumb.cuh -- warp-per-image kernel for 1/8-scale decodes of small
// images (thumbnails; BASELINE c4: 161x161 -> 1/8 -> 64x64, batch 4096).
//
// At scale 1/8 a block decodes to one sample: its DC (reading R1), so a
// 161x161 image is a 21x21 luma + 11x11 chroma picture and the work is the
// 64x64x3 output.  The tiled kernel spends most of such a CTA's life in
// barrier-separated phases with global-latency round trips between them;
// here one warp owns one image end to end (no CTA barriers, only __syncwarp),
// many images per SM are in flight, and the kernel is bound by the output
// stores.  Same arithmetic as the tiled kernel for every u8 step (DC round,
// 4:2:0 triangle upsample, exact colour) and the same packed fp32 bilinear +
// normalize, so its outputs are bit-identical to the tiled kernel's.
#pragma once
#include "smol_kernels.cuh"

namespace smol {

constexpr int kThumbWarps = 4;                 // images in flight per CTA
constexpr int kThumbMaxFoot = 32;              // decoded luma footprint limit (px per side)
constexpr int kThumbMaxOut = 128;              // output width / height limit
constexpr int kThumbCP = kThumbMaxFoot / 2 + 2;   // chroma footprint pitch
struct ThumbWarpSmem {
  uint32_t rgb[kThumbMaxFoot * kThumbMaxFoot + 1];  // RGBx of the luma footprint (+1: x0 + 1 read at the end)
  uint8_t y[kThumbMaxFoot * kThumbMaxFoot];
  uint8_t c[2][kThumbCP * kThumbCP];
  int4 xp[kThumbMaxOut / 2];                     // per output column pair: {4 x0 (a), 4 x0 (b), w (a), w (b)}
  int2 yt[kThumbMaxOut];                         // per output row:    {y0 - ly0 | (y1 - ly0) << 16, w}
  TileLayout L;
};
constexpr int kThumbSmem = kThumbWarps * (int)sizeof(ThumbWarpSmem);

template <bool F16, bool PACKED>
__global__ void __launch_bounds__(kThumbWarps * 32) smol_thumb_kernel(const __grid_constant__ KParams kp,
                                                                      int n_images) {
  extern __shared__ __align__(16) uint8_t tsm[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  ThumbWarpSmem& S = reinterpret_cast<ThumbWarpSmem*>(tsm)[warp];
  constexpr int E = PACKED ? 1 : 64;            // DC at element 0 of a stored block
  using OutT = typename std::conditional<F16, __half, float>::type;
  const int OW = kp.OW, OH = kp.OH;
  const uint32_t plane = (uint32_t)OW * OH;
  for (int n = blockIdx.x * kThumbWarps + warp; n < n_images; n += gridDim.x * kThumbWarps) {
    const DevRef ref = kp.refs[n];
    DevImage im = kp.kinds[ref.kind];
    im.coef[0] = ref.coef[0]; im.coef[1] = ref.coef[1]; im.coef[2] = ref.coef[2];
    if (kp.lays) {                                // precomputed per image kind: the warp copies it in
      static_assert(sizeof(TileLayout) % 4 == 0, "TileLayout copied in 4-byte words");
      const uint32_t* src = reinterpret_cast<const uint32_t*>(kp.lays + ref.kind * kp.lay_stride);
      uint32_t* dst = reinterpret_cast<uint32_t*>(&S.L);
      for (int i = lane; i < (int)(sizeof(TileLayout) / 4); i += 32) dst[i] = __ldg(src + i);
    } else if (lane == 0) {
      tile_layout(im, 8, 0, OH, 0, OW, S.L, kYPTiny);
    }
    __syncwarp();
    const int lx0 = S.L.lx0, ly0 = S.L.ly0, fw = S.L.lx1 - lx0 + 1, fh = S.L.ly1 - ly0 + 1;
    const int cx0 = S.L.cx0, cy0 = S.L.cy0, cw = S.L.cx1 - cx0 + 1, ch = S.L.cy1 - cy0 + 1;
    // magic-number divisions by the runtime widths (all operands < 2^16)
    const FastDiv fd_fw = S.L.fd_fw, fd_cw = S.L.fd_cw;   // (precomputed with the layout)
    // taps (reading R9: exact integers); a clamped upper tap gets weight 0
    // column taps per output pair, byte offsets of x0 in an RGB row; the
    // kernel always reads x0 + 1 (a clamped upper tap has weight 0, and the
    // byte -> float trick keeps even stale words finite)
    // (precomputed once per image kind by the host when it could: copied in)
    if (S.L.tap_off >= 0) {
      const int4* src = kp.taps + S.L.tap_off;
      const int nxp = (OW + 1) >> 1;
      for (int q = lane; q < nxp; q += 32) S.xp[q] = src[q];
      for (int i = lane; i < (OH + 1) >> 1; i += 32) reinterpret_cast<int4*>(S.yt)[i] = src[nxp + i];
    } else {
      for (int q = lane; q < (OW + 1) >> 1; q += 32) thumb_xp(im, S.L, OW, q, reinterpret_cast<int*>(&S.xp[q]));
      for (int i = lane; i < OH; i += 32) thumb_yt(im, S.L, i, reinterpret_cast<int*>(&S.yt[i]));
    }
    // 1/8 decode (reading R1/R3): u8 = clamp(floor(DC * Q0 / 8 + 128 + 1/2))
    const float qy = (float)kp.qtables[im.qidx[0] * 64] * 0.125f;
    for (int p = lane; p < fw * fh; p += 32) {
      const int r = (int)fdiv((uint32_t)p, fd_fw), x = p - r * fw;
      const int16_t dc = __ldg(im.coef[0] + (size_t)(ly0 + r) * im.stride[0] + (size_t)(lx0 + x) * E);
      S.y[r * kThumbMaxFoot + x] = (uint8_t)round_u8((float)dc * qy);
    }
    for (int cc = 0; cc < 2; ++cc) {
      const float qc = (float)kp.qtables[im.qidx[1 + cc] * 64] * 0.125f;
      for (int p = lane; p < cw * ch; p += 32) {
        const int r = (int)fdiv((uint32_t)p, fd_cw), x = p - r * cw;
        uint8_t v = 128;                          // grayscale: neutral chroma (reading R14)
        if (!im.gray) {
          const int16_t dc = __ldg(im.coef[1 + cc] + (size_t)(cy0 + r) * im.stride[1 + cc] + (size_t)(cx0 + x) * E);
          v = (uint8_t)round_u8((float)dc * qc);
        }
        S.c[cc][r * kThumbCP + x] = v;
      }
    }
    __syncwarp();
    // 4:2:0 centred triangle upsample (reading R2, neighbours clamped to the
    // valid chroma size) + exact JFIF colour (R6)
    for (int p = lane; p < fw * fh; p += 32) {
      const int r = (int)fdiv((uint32_t)p, fd_fw), x = p - r * fw;
      const int X = lx0 + x, Yr = ly0 + r;
      const int i = X >> 1, j = Yr >> 1;
      const int in = min(max((X & 1) ? i + 1 : i - 1, 0), im.Wc - 1);
      const int jn = min(max((Yr & 1) ? j + 1 : j - 1, 0), im.Hc - 1);
      const int a = (j - cy0) * kThumbCP, b = (jn - cy0) * kThumbCP;
      const int ci = i - cx0, cn = in - cx0;
      const int cb = 9 * S.c[0][a + ci] + 3 * S.c[0][a + cn] + 3 * S.c[0][b + ci] + S.c[0][b + cn];
      const int cr = 9 * S.c[1][a + ci] + 3 * S.c[1][a + cn] + 3 * S.c[1][b + ci] + S.c[1][b + cn];
      S.rgb[r * kThumbMaxFoot + x] = colour(S.y[r * kThumbMaxFoot + x], cb, cr);
    }
    __syncwarp();
    // bilinear (reading R8) + normalize: the warp walks the output rows
    // together, lane l holding output pixel pairs l and l + 32 (2 pixels per
    // packed FP32x2 instruction); u8 -> float by one PRMT into the 2^23
    // magic (the bias cancels in b - a) -- the tiled kernel's formulation, so
    // the outputs are bit-identical to it.  All lanes share each row's taps,
    // so the horizontal lerps of a source row are recomputed only where the
    // row taps move (thumbnails magnify: 21 -> 64 rows at c4), by the whole
    // warp at once; the old bottom becomes the new top when they move down
    // one row (bit-identical).
    OutT* const outn = reinterpret_cast<OutT*>(kp.out) + (size_t)n * 3 * plane;
    const uint32_t magic = kp.magic;
    const float2 na0 = f2(kp.na[0]), na1 = f2(kp.na[1]), na2 = f2(kp.na[2]);
    const float2 nb0 = f2(kp.nb[0]), nb1 = f2(kp.nb[1]), nb2 = f2(kp.nb[2]);
    const int npair = (OW + 1) >> 1;              // <= kThumbMaxOut / 2 = 64: two pairs per lane at most
    const bool has1 = lane + 32 < npair;
    const int4 tx0 = S.xp[min(lane, npair - 1)];
    const int4 tx1 = S.xp[min(lane + 32, npair - 1)];
    float2 T0[3], B0[3], T1[3], B1[3];            // horizontal lerps of the top / bottom source rows [ch]
    auto hlerp = [&](int row, const int4& tx, float2 (&H)[3]) {
      const uint8_t* base = reinterpret_cast<const uint8_t*>(S.rgb + row * kThumbMaxFoot);
      const float2 wx = make_float2(__int_as_float(tx.z), __int_as_float(tx.w));
      const uint32_t p0 = lds_u32(base + tx.x), p1 = lds_u32(base + tx.x + 4);
      const uint32_t q0 = lds_u32(base + tx.y), q1 = lds_u32(base + tx.y + 4);
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        const int sel = 0x7540 + c;
        const float2 fa = make_float2(__uint_as_float(__byte_perm(p0, magic, sel)), __uint_as_float(__byte_perm(q0, magic, sel)));
        const float2 fb = make_float2(__uint_as_float(__byte_perm(p1, magic, sel)), __uint_as_float(__byte_perm(q1, magic, sel)));
        H[c] = __ffma2_rn(wx, __ffma2_rn(fa, f2(-1.f), fb), __fadd2_rn(fa, f2(-8388608.f)));
      }
    };
    const bool vec = (OW & 1) == 0 && kp.out_vec;  // pixel pairs 8-B (f32) / 4-B (f16) aligned
    auto store = [&](OutT* o, const float2 (&T)[3], const float2 (&B)[3], float2 wy2, int x) {
      float2 v[3];
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        const float2 vv = __ffma2_rn(wy2, __ffma2_rn(T[c], f2(-1.f), B[c]), T[c]);
        v[c] = __ffma2_rn(vv, c == 0 ? na0 : c == 1 ? na1 : na2, c == 0 ? nb0 : c == 1 ? nb1 : nb2);
      }
      if (vec) {
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          if constexpr (F16) {
            const __half2 h = __floats2half2_rn(v[c].x, v[c].y);
            __stcs(reinterpret_cast<uint32_t*>(o + c * plane), *reinterpret_cast<const uint32_t*>(&h));
          } else {
            __stcs(reinterpret_cast<float2*>(o + c * plane), v[c]);
          }
        }
      } else {
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          if constexpr (F16) {
            o[c * plane] = __float2half_rn(v[c].x);
            if (x + 1 < OW) o[1 + c * plane] = __float2half_rn(v[c].y);
          } else {
            o[c * plane] = v[c].x;
            if (x + 1 < OW) o[1 + c * plane] = v[c].y;
          }
        }
      }
    };
    int c0 = -1, c1 = -1;                         // source rows of T and B (uniform over the warp)
    const bool has0 = lane < npair;
#pragma unroll 1
    for (int oy = 0; oy < OH; ++oy) {
      const int2 ty = S.yt[oy];
      const int i0 = ty.x & 0xffff, i1 = ty.x >> 16;
      if (i0 != c0 || i1 != c1) {
        if (i0 == c1) {
#pragma unroll
          for (int c = 0; c < 3; ++c) { T0[c] = B0[c]; T1[c] = B1[c]; }
        } else {
          hlerp(i0, tx0, T0);
          if (has1) hlerp(i0, tx1, T1);
        }
        hlerp(i1, tx0, B0);
        if (has1) hlerp(i1, tx1, B1);
        c0 = i0; c1 = i1;
      }
      const float2 wy2 = f2(__int_as_float(ty.y));
      OutT* const orow = outn + (uint32_t)oy * OW;
      if (has0) store(orow + 2 * lane, T0, B0, wy2, 2 * lane);
      if (has1) store(orow + 2 * (lane + 32), T1, B1, wy2, 2 * (lane + 32));
    }
    __syncwarp();                                 // smem reused by the warp's next image
  }
}

}  // namespace smol
