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
constexpr int kThumbRun = 8;                   // output rows per lane task (row-run reuse; 16 / 32 no gain, r02t)
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
    const FastDiv fd_fw = S.L.fd_fw, fd_cw = S.L.fd_cw, fd_nq = S.L.fd_q4;   // (precomputed with the layout)
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
    // bilinear (reading R8) + normalize, 4 consecutive output pixels per lane,
    // two pixels per packed FP32x2 instruction; u8 -> float by one PRMT into
    // the 2^23 magic (the bias cancels in b - a) -- the tiled kernel's
    // formulation, so the outputs are bit-identical to it
    OutT* const outn = reinterpret_cast<OutT*>(kp.out) + (size_t)n * 3 * plane;
    const int nq = (OW + 3) >> 2;
    const uint32_t magic = kp.magic;
    const float2 na0 = f2(kp.na[0]), na1 = f2(kp.na[1]), na2 = f2(kp.na[2]);
    const float2 nb0 = f2(kp.nb[0]), nb1 = f2(kp.nb[1]), nb2 = f2(kp.nb[2]);
    // a lane walks one 4-pixel column quad down a run of kThumbRun rows:
    // the horizontal lerps of a source row are reused while the row taps
    // stay put (thumbnails magnify: 21 -> 64 rows at c4), the old bottom
    // becomes the new top when they move down one row (bit-identical)
    const int ngr = (OH + kThumbRun - 1) / kThumbRun;
    for (int t = lane; t < nq * ngr; t += 32) {
      const int g = (int)fdiv((uint32_t)t, fd_nq), q = t - g * nq, ox = 4 * q;
      const int ra = g * kThumbRun, rb = min(ra + kThumbRun, OH);
      const int4 txa = S.xp[min(ox >> 1, ((OW + 1) >> 1) - 1)];
      const int4 txb = S.xp[min((ox + 2) >> 1, ((OW + 1) >> 1) - 1)];
      float2 T[3][2], B[3][2];
      auto hlerp = [&](int row, float2 (&H)[3][2]) {
        const uint8_t* base = reinterpret_cast<const uint8_t*>(S.rgb + row * kThumbMaxFoot);
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int4 tx = e == 0 ? txa : txb;
          const float2 wx = make_float2(__int_as_float(tx.z), __int_as_float(tx.w));
          const uint32_t p0 = lds_u32(base + tx.x), p1 = lds_u32(base + tx.x + 4);
          const uint32_t q0 = lds_u32(base + tx.y), q1 = lds_u32(base + tx.y + 4);
#pragma unroll
          for (int c = 0; c < 3; ++c) {
            const int sel = 0x7540 + c;
            const float2 fa = make_float2(__uint_as_float(__byte_perm(p0, magic, sel)), __uint_as_float(__byte_perm(q0, magic, sel)));
            const float2 fb = make_float2(__uint_as_float(__byte_perm(p1, magic, sel)), __uint_as_float(__byte_perm(q1, magic, sel)));
            H[c][e] = __ffma2_rn(wx, __ffma2_rn(fa, f2(-1.f), fb), __fadd2_rn(fa, f2(-8388608.f)));
          }
        }
      };
      int c0 = -1, c1 = -1;                       // source rows of T and B
      OutT* o = outn + (uint32_t)ra * OW + ox;    // walks down the run
#pragma unroll 1
      for (int oy = ra; oy < rb; ++oy, o += OW) {
        const int2 ty = S.yt[oy];
        const int i0 = ty.x & 0xffff, i1 = ty.x >> 16;
        if (i0 != c0 || i1 != c1) {
          if (i0 == c1) {
#pragma unroll
            for (int c = 0; c < 3; ++c) { T[c][0] = B[c][0]; T[c][1] = B[c][1]; }
          } else {
            hlerp(i0, T);
          }
          hlerp(i1, B);
          c0 = i0; c1 = i1;
        }
        const float2 wy2 = f2(__int_as_float(ty.y));
        float v[3][4];
#pragma unroll
        for (int c = 0; c < 3; ++c)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const float2 vv = __ffma2_rn(wy2, __ffma2_rn(T[c][e], f2(-1.f), B[c][e]), T[c][e]);
            const float2 yn = __ffma2_rn(vv, c == 0 ? na0 : c == 1 ? na1 : na2, c == 0 ? nb0 : c == 1 ? nb1 : nb2);
            v[c][2 * e] = yn.x;
            v[c][2 * e + 1] = yn.y;
          }
        if ((OW & 3) == 0 && kp.out_vec) {
#pragma unroll
          for (int c = 0; c < 3; ++c) {
            if constexpr (F16) {
              const __half2 h0 = __floats2half2_rn(v[c][0], v[c][1]), h1 = __floats2half2_rn(v[c][2], v[c][3]);
              uint2 u;
              u.x = *reinterpret_cast<const uint32_t*>(&h0);
              u.y = *reinterpret_cast<const uint32_t*>(&h1);
              __stcs(reinterpret_cast<uint2*>(o + c * plane), u);
            } else {
              __stcs(reinterpret_cast<float4*>(o + c * plane), make_float4(v[c][0], v[c][1], v[c][2], v[c][3]));
            }
          }
        } else {
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            if (ox + e >= OW) break;
#pragma unroll
            for (int c = 0; c < 3; ++c) {
              if constexpr (F16) o[e + c * plane] = __float2half_rn(v[c][e]);
              else o[e + c * plane] = v[c][e];
            }
          }
        }
      }
    }
    __syncwarp();                                 // smem reused by the warp's next image
  }
}

}  // namespace smol
