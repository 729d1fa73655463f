// smol_kernels.cuh -- the fused sm_100a kernel of the Smol preprocessing hot
// path: dequantize -> scaled IDCT -> u8 -> 4:2:0 upsample -> YCbCr->RGB ->
// bilinear resize + crop -> normalize -> NCHW.  One CTA per (image, output
// tile); decoded pixels live only in shared memory.
//
// Each CTA walks its tile's decoded-row footprint in 16-row steps (one MCU
// row at scale 1) with rolling shared-memory windows, so every coefficient
// block under the footprint is read and transformed once per tile:
//   IDCT(0)                                                          sync
//   step s:  L2 bulk prefetch of step s+1's ROI block rows
//            colour RGB rows (ready_{s-1}, ready_s]: 2x4-pixel tasks, 4:2:0
//                   triangle upsample + exact JFIF -> packed RGBx ring   sync
//            IDCT(s+1): thread per block, warp-uniform pruning of all-zero
//                   high rows -> u8 Y / Cb / Cr rings
//            + output of every output row whose lower tap row is ready:
//                   bilinear + FMA normalize, 4 pixels per task, NCHW
//                   streaming stores                                    sync
#pragma once
#include <cuda_fp16.h>
#include <stdint.h>
#include <type_traits>
#include <cstddef>

#include "smol_geom.cuh"

// Output-phase scheduling (measured, profiles/r01h_output_schedule.md): at
// scale 1 the output tasks share the phase with the next step's IDCT and are
// grabbed dynamically, two per lane per grab, interleaved by the compiler; at
// scales 1/2..1/8 that IDCT is small and a static stride wins.
#ifndef SMOL_OUT_PER_GRAB
#define SMOL_OUT_PER_GRAB 2      // scale 1: output tasks per lane per work-counter grab
#endif
#ifndef SMOL_OUT_STATIC
#define SMOL_OUT_STATIC 2        // 0: dynamic everywhere; 1: static everywhere; 2: static at scales 1/2..1/8
#endif

namespace smol {


// Basis constants, computed on the host in double from their definitions
// (smol_preproc.cu: init_basis) and uploaded once per device.
//   t[u][x]  = sqrt2 C(u) cos((2x+1) u pi/16), x < 4   (t[0][x] = 1, t[4][x] = +-1 exactly)
//   a2[j][u] = 1/2 sum_{x=2j}^{2j+1} t[u][x], j < 2    (a2[j][0] = 1, a2[j][4] = 0 exactly)
//   a4[u]    = 1/4 sum_{x=0}^{3} t[u][x]               (a4[0] = 1; 0 for u = 2, 4, 6)
// Output j and P-1-j are mirror images: t[u][7-x] = (-1)^u t[u][x] (same for a_k).
// Colour: kR, kB = fl32(1.402/16), fl32(1.772/16); cR, cB = fl32(1/2 - 2048 kR),
// fl32(1/2 - 2048 kB) + 2^-13 (see colour()).
struct Basis {
  float t[8][4];
  float a2[2][8];
  float a4[8];
  float kR, kB, cR, cB;
  uint32_t gK1, gCb, gCr;          // G = Y + (gK1 + gCb cb16 + gCr cr16) / 2e6 - 136 (mod 2^32; see colour())
  float2 tp[4][4];   // column pass pairs: tp[k][y] = (t[2k][y], t[2k+1][y])
};

// One copy per translation unit (internal linkage; the library is built
// without relocatable device code): every TU that instantiates kernels
// exports an upload function (smol_launch.h) and the runtime fills all.
namespace {
__constant__ Basis c_basis;
}

// ------------------------------------------------------------ 1-D IDCTs ---
// Reading R1 (Definition A), separable form of the oracle's sum.  The
// scale-1 basis t(u,x) = sqrt2 C(u) cos((2x+1) u pi/16) is compiled in as
// immediates (FFMA immediate form; init_basis checks these literals against
// the double-precision formula at plan creation):  c_k = sqrt2 cos(k pi/16).
constexpr float kC1 = 1.387039845322f, kC2 = 1.306562964876f, kC3 = 1.175875602419f,
                kC5 = 0.785694958387f, kC6 = 0.541196100146f, kC7 = 0.275899379283f;
__host__ __device__ constexpr float basis_t(int u, int x) {
  // t(u, x) for x < 4 (t(u, 7-x) = (-1)^u t(u, x)); t(0,x) = 1, t(4,x) = +-1 exactly
  return u == 0 ? 1.f
       : u == 1 ? (x == 0 ? kC1 : x == 1 ? kC3 : x == 2 ? kC5 : kC7)
       : u == 2 ? (x == 0 ? kC2 : x == 1 ? kC6 : x == 2 ? -kC6 : -kC2)
       : u == 3 ? (x == 0 ? kC3 : x == 1 ? -kC7 : x == 2 ? -kC1 : -kC5)
       : u == 4 ? ((x == 0 || x == 3) ? 1.f : -1.f)
       : u == 5 ? (x == 0 ? kC5 : x == 1 ? -kC1 : x == 2 ? kC7 : kC3)
       : u == 6 ? (x == 0 ? kC6 : x == 1 ? -kC2 : x == 2 ? kC2 : -kC6)
       :          (x == 0 ? kC7 : x == 1 ? -kC5 : x == 2 ? kC3 : -kC1);
}

// 8-point IDCT, inputs u >= W known zero (compile time).  The FMA chains
// start from d[0] (weight exactly 1) and the exact +-1 entries of u = 4, so
// DC-only and {0,4}-only inputs are transformed exactly (reading R3).
template <int W>
__device__ __forceinline__ void idct8(const float (&d)[8], float (&o)[8]) {
#pragma unroll
  for (int x = 0; x < 4; ++x) {
    float e = d[0];
    if (W > 4) e = (x == 0 || x == 3) ? e + d[4] : e - d[4];
    if (W > 2) e = fmaf(d[2], basis_t(2, x), e);
    if (W > 6) e = fmaf(d[6], basis_t(6, x), e);
    float od = 0.f;
    if (W > 1) od = d[1] * basis_t(1, x);
    if (W > 3) od = fmaf(d[3], basis_t(3, x), od);
    if (W > 5) od = fmaf(d[5], basis_t(5, x), od);
    if (W > 7) od = fmaf(d[7], basis_t(7, x), od);
    if (W > 1) { o[x] = e + od; o[7 - x] = e - od; }
    else { o[x] = e; o[7 - x] = e; }
  }
}

__device__ __forceinline__ void idct4(const float (&d)[8], float (&o)[4]) {
#pragma unroll
  for (int j = 0; j < 2; ++j) {
    float e = fmaf(d[2], c_basis.a2[j][2], d[0]);
    e = fmaf(d[6], c_basis.a2[j][6], e);
    float od = d[1] * c_basis.a2[j][1];
    od = fmaf(d[3], c_basis.a2[j][3], od);
    od = fmaf(d[5], c_basis.a2[j][5], od);
    od = fmaf(d[7], c_basis.a2[j][7], od);
    o[j] = e + od;
    o[3 - j] = e - od;
  }
}

__device__ __forceinline__ void idct2(const float (&d)[8], float (&o)[2]) {
  float od = d[1] * c_basis.a4[1];
  od = fmaf(d[3], c_basis.a4[3], od);
  od = fmaf(d[5], c_basis.a4[5], od);
  od = fmaf(d[7], c_basis.a4[7], od);
  o[0] = d[0] + od;
  o[1] = d[0] - od;
}

// idct4 / idct2 of two rows at once (lane .x, lane .y), FP32x2 packed: the
// same IEEE operations in the same order as the scalar forms (e - od as
// e + (-1)(od), exact product, one rounding), so bit-identical.
__device__ __forceinline__ float2 f2c(float a) { return make_float2(a, a); }
__device__ __forceinline__ void idct4x2(const float2 (&d)[8], float2 (&o)[4]) {
#pragma unroll
  for (int j = 0; j < 2; ++j) {
    float2 e = __ffma2_rn(d[2], f2c(c_basis.a2[j][2]), d[0]);
    e = __ffma2_rn(d[6], f2c(c_basis.a2[j][6]), e);
    float2 od = __fmul2_rn(d[1], f2c(c_basis.a2[j][1]));
    od = __ffma2_rn(d[3], f2c(c_basis.a2[j][3]), od);
    od = __ffma2_rn(d[5], f2c(c_basis.a2[j][5]), od);
    od = __ffma2_rn(d[7], f2c(c_basis.a2[j][7]), od);
    o[j] = __fadd2_rn(e, od);
    o[3 - j] = __ffma2_rn(od, f2c(-1.f), e);
  }
}
__device__ __forceinline__ void idct2x2(const float2 (&d)[8], float2 (&o)[2]) {
  float2 od = __fmul2_rn(d[1], f2c(c_basis.a4[1]));
  od = __ffma2_rn(d[3], f2c(c_basis.a4[3]), od);
  od = __ffma2_rn(d[5], f2c(c_basis.a4[5]), od);
  od = __ffma2_rn(d[7], f2c(c_basis.a4[7]), od);
  o[0] = __fadd2_rn(d[0], od);
  o[1] = __ffma2_rn(od, f2c(-1.f), d[0]);
}

// Reading R3: clamp(floor(v + 128 + 1/2), 0, 255) in one F2I.U8.FLOOR (cvt
// saturates to the u8 range).
__device__ __forceinline__ uint32_t round_u8(float v) {
  uint32_t r;
  asm("cvt.rmi.sat.u8.f32 %0, %1;" : "=r"(r) : "f"(v + 128.5f));
  return r;
}
__device__ __forceinline__ uint32_t floor_u8(float v) {
  uint32_t r;
  asm("cvt.rmi.sat.u8.f32 %0, %1;" : "=r"(r) : "f"(v));
  return r;
}

__device__ __forceinline__ float lo16f(int x) { return (float)(int16_t)(x & 0xffff); }
__device__ __forceinline__ void unpack_row(const int4 r, float (&d)[8]) {
  d[0] = lo16f(r.x); d[1] = (float)(r.x >> 16);
  d[2] = lo16f(r.y); d[3] = (float)(r.y >> 16);
  d[4] = lo16f(r.z); d[5] = (float)(r.z >> 16);
  d[6] = lo16f(r.w); d[7] = (float)(r.w >> 16);
}

__device__ __forceinline__ uint32_t pack4(uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
  return __byte_perm(__byte_perm(a, b, 0x0040), __byte_perm(c, d, 0x0040), 0x5410);
}

// Full-scale block, row pass: rows v < HR (rows >= HR are all-zero in the
// whole warp), inputs u < W.  Level shift and rounding offset (+128 + 1/2,
// reading R3) ride on the DC term: t(0, .) = 1 exactly, so adding it to
// D(0,0) adds it to every output sample.
// Packed FP32x2 (FFMA2/FADD2, sm_100): two independent IEEE fp32 operations
// per instruction, bitwise identical to the scalar ones.
__device__ __forceinline__ float2 f2(float a) { return make_float2(a, a); }

// 8-point IDCT of two rows at once (lane .x = row v, .y = row v+1); same
// operation order as idct8 (exact DC / u=4 paths preserved).
template <int W>
__device__ __forceinline__ void idct8x2(const float2 (&d)[8], float2 (&o)[8]) {
#pragma unroll
  for (int x = 0; x < 4; ++x) {
    float2 e = d[0];
    if (W > 4) e = (x == 0 || x == 3) ? __fadd2_rn(e, d[4]) : __ffma2_rn(d[4], f2(-1.f), e);
    if (W > 2) e = __ffma2_rn(d[2], f2(basis_t(2, x)), e);
    if (W > 6) e = __ffma2_rn(d[6], f2(basis_t(6, x)), e);
    float2 od = f2(0.f);
    if (W > 1) od = __fmul2_rn(d[1], f2(basis_t(1, x)));
    if (W > 3) od = __ffma2_rn(d[3], f2(basis_t(3, x)), od);
    if (W > 5) od = __ffma2_rn(d[5], f2(basis_t(5, x)), od);
    if (W > 7) od = __ffma2_rn(d[7], f2(basis_t(7, x)), od);
    if (W > 1) { o[x] = __fadd2_rn(e, od); o[7 - x] = __ffma2_rn(od, f2(-1.f), e); }
    else { o[x] = e; o[7 - x] = e; }
  }
}

// Full-scale block, row pass: rows v < HR (rows >= HR are all-zero in the
// whole warp), inputs u < W, two rows per packed instruction.  Level shift
// and rounding offset (+128 + 1/2, reading R3) ride on the DC term:
// t(0, .) = 1 exactly, so adding it to D(0,0) adds it to every sample.
template <int W, int HR>
__device__ __forceinline__ void idct_rows(const int4 (&raw)[8], const float* q, float (&m)[8][8]) {
#pragma unroll
  for (int v = 0; v < HR; v += 2) {
    float a[8], b[8];
    unpack_row(raw[v], a);
    unpack_row(raw[v + 1], b);
    const float4 qa0 = *reinterpret_cast<const float4*>(q + v * 8);
    const float4 qa1 = *reinterpret_cast<const float4*>(q + v * 8 + 4);
    const float4 qb0 = *reinterpret_cast<const float4*>(q + v * 8 + 8);
    const float4 qb1 = *reinterpret_cast<const float4*>(q + v * 8 + 12);
    float2 d[8];
    d[0] = make_float2(a[0] * qa0.x, b[0] * qb0.x); d[1] = make_float2(a[1] * qa0.y, b[1] * qb0.y);
    d[2] = make_float2(a[2] * qa0.z, b[2] * qb0.z); d[3] = make_float2(a[3] * qa0.w, b[3] * qb0.w);
    d[4] = make_float2(a[4] * qa1.x, b[4] * qb1.x); d[5] = make_float2(a[5] * qa1.y, b[5] * qb1.y);
    d[6] = make_float2(a[6] * qa1.z, b[6] * qb1.z); d[7] = make_float2(a[7] * qa1.w, b[7] * qb1.w);
    if (v == 0) d[0].x += 128.5f;
    float2 o[8];
    idct8x2<W>(d, o);
#pragma unroll
    for (int x = 0; x < 8; ++x) { m[v][x] = o[x].x; m[v + 1][x] = o[x].y; }
  }
}

template <int H>
__device__ __forceinline__ void idct_cols(const float (&m)[8][8], uint32_t (&px)[8][2]) {
  // column x's bytes are merged into the row words as they are produced
  // (one PRMT per byte; keeps the live set at m + px)
#pragma unroll
  for (int x = 0; x < 8; ++x) {
    float col[8], f[8];
#pragma unroll
    for (int v = 0; v < 8; ++v) col[v] = (v < H) ? m[v][x] : 0.f;
    idct8<H>(col, f);
#pragma unroll
    for (int y = 0; y < 8; ++y) {
      const uint32_t b = floor_u8(f[y]);
      uint32_t& w = px[y][x >> 2];
      if ((x & 3) == 0) w = b;
      else w = __byte_perm(w, b, (x & 3) == 1 ? 0x3240 : (x & 3) == 2 ? 0x3410 : 0x4210);
    }
  }
}

// Coefficient-block layouts (smol_preproc.h smol_coef_layout).  DENSE64:
// 64 int16 per block, natural order.  PACKED: only the coefficients whose
// box-averaged basis a_k(u, .) is not identically zero at scale 1/K (reading
// R1), row-major over the index set, padded to 8 bytes:
//   K=2: u,v in {0,1,2,3,5,6,7}  49 -> 52 int16 (104 B)
//   K=4: u,v in {0,1,3,5,7}      25 -> 28 int16 ( 56 B)
//   K=8: DC only                  1 int16      (  2 B)
// Definition B (reading R16, plan option SMOL_IDCT_TRUNCATED) uses only the
// top-left N x N coefficients (N = 8/K); its PACKED blocks hold exactly
// those, row-major: K=2: 16 int16 (32 B), K=4: 4 int16 (8 B), K=8: DC.
template <int K, bool PACKED, bool DB = false>
struct BlockFmt {
  static constexpr int kElems = !PACKED ? 64
                              : DB ? (8 / K) * (8 / K)
                                   : (K == 1 ? 64 : K == 2 ? 52 : K == 4 ? 28 : 1);
};
__host__ __device__ constexpr int packed_set(int K, int i) {   // i-th index of the K's set
  return K == 2 ? (i < 4 ? i : i + 1) : K == 4 ? (i == 0 ? 0 : 2 * i - 1) : i;
}
__host__ __device__ constexpr int packed_n(int K) { return K == 2 ? 7 : K == 4 ? 5 : K == 8 ? 1 : 8; }

template <int NWORDS>
__device__ __forceinline__ float half_of(const uint32_t (&w)[NWORDS], int e) {
  return (e & 1) ? (float)((int)w[e >> 1] >> 16) : (float)(int16_t)(w[e >> 1] & 0xffff);
}

// Decode one block at scale 1/K: px[y] holds the P samples of output row y
// (little-endian bytes, 2 words per row at K = 1).  `act` = this lane has a
// block; every lane of the warp must call it (warp reductions pick the
// nonzero row extent).
// Definition B, N = 8/K: N-point IDCT with b_N(u,x) = sqrt2 C(u)
// cos((2x+1) u pi / 2N): b_4(1,.) = (c2, c6, -c6, -c2), b_4(3,.) = (c6, -c2,
// c2, -c6) (c_k = sqrt2 cos(k pi/16) of the 8-point basis), b_4(2,.) =
// (1,-1,-1,1) and b_2(1,.) = (1,-1) exactly, so DC and u = N/2 inputs are
// transformed exactly (reading R3).
template <int N>
__device__ __forceinline__ void idct_trunc(const float (&d)[N], float (&o)[N]) {
  if constexpr (N == 4) {
    const float e0 = d[0] + d[2], e1 = d[0] - d[2];
    const float od0 = fmaf(d[3], kC6, d[1] * kC2);
    const float od1 = fmaf(d[3], -kC2, d[1] * kC6);
    o[0] = e0 + od0; o[3] = e0 - od0;
    o[1] = e1 + od1; o[2] = e1 - od1;
  } else {
    o[0] = d[0] + d[1];
    o[1] = d[0] - d[1];
  }
}

template <int K, bool PACKED, bool DB = false>
__device__ __forceinline__ void decode_block(bool act, const int16_t* src, const float* q,
                                             uint32_t (&px)[8][2]) {
  constexpr int P = 8 / K;
  if constexpr (DB && (K == 2 || K == 4)) {
    // Definition B (reading R16): P-point IDCT of the top-left P x P
    // coefficients (Q/8 folded in q: v = 1/8 sum D b_P b_P)
    float g[P][P];
#pragma unroll
    for (int v = 0; v < P; ++v) {
      float d[P];
      if constexpr (K == 2) {
        const int2 r = act ? __ldg(reinterpret_cast<const int2*>(src + (PACKED ? 4 * v : 8 * v))) : make_int2(0, 0);
        d[0] = (float)(int16_t)(r.x & 0xffff); d[1] = (float)(r.x >> 16);
        d[2] = (float)(int16_t)(r.y & 0xffff); d[3] = (float)(r.y >> 16);
      } else {
        const int r = act ? __ldg(reinterpret_cast<const int*>(src + (PACKED ? 2 * v : 8 * v))) : 0;
        d[0] = (float)(int16_t)(r & 0xffff); d[1] = (float)(r >> 16);
      }
#pragma unroll
      for (int u = 0; u < P; ++u) d[u] *= q[v * 8 + u];
      if (v == 0) d[0] += 128.5f;           // level shift + rounding offset (b_P(0, .) = 1 exactly)
      idct_trunc<P>(d, g[v]);
    }
#pragma unroll
    for (int x = 0; x < P; ++x) {
      float col[P], f[P];
#pragma unroll
      for (int v = 0; v < P; ++v) col[v] = g[v][x];
      idct_trunc<P>(col, f);
#pragma unroll
      for (int y = 0; y < P; ++y) {
        const uint32_t b = floor_u8(f[y]);
        px[y][0] = (x == 0) ? b : (px[y][0] | (b << (8 * x)));
      }
    }
  } else if constexpr (K == 8) {
    px[0][0] = act ? round_u8((float)__ldg(src) * q[0]) : 0u;
  } else if constexpr (K == 1) {
    int4 raw[8];
#pragma unroll
    for (int v = 0; v < 8; ++v)
      raw[v] = act ? __ldg(reinterpret_cast<const int4*>(src) + v) : make_int4(0, 0, 0, 0);
    uint32_t rows = 0;
#pragma unroll
    for (int v = 0; v < 8; ++v) rows |= ((raw[v].x | raw[v].y | raw[v].z | raw[v].w) != 0) << v;
    // prune by the warp's highest nonzero coefficient row (one code variant
    // per extent: more variants cost more in I-cache misses than they save)
    const int H = (int)__reduce_max_sync(0xffffffffu, 32 - __clz(rows));
    // (a column pass on FFMA2 row pairs, and both passes on packed column
    // pairs, measured no faster: r02 A/B)
    float m[8][8];
    if (H <= 6) { idct_rows<8, 6>(raw, q, m); idct_cols<6>(m, px); }
    else { idct_rows<8, 8>(raw, q, m); idct_cols<8>(m, px); }
  } else {
    // K = 2 (4x4 out, u,v != 4) and K = 4 (2x2 out, u,v in {0,1,3,5,7}):
    // rows/columns outside the index set have an exactly-zero basis.
    constexpr int NS = packed_n(K);
    float g[8][P];
#pragma unroll
    for (int v = 0; v < 8; ++v)
#pragma unroll
      for (int j = 0; j < P; ++j) g[v][j] = 0.f;
    constexpr int NW = PACKED ? BlockFmt<K, true>::kElems / 4 : 1;   // 8-byte words
    uint32_t w[2 * NW];
    if constexpr (PACKED) {
#pragma unroll
      for (int i = 0; i < NW; ++i) {
        const int2 t = act ? __ldg(reinterpret_cast<const int2*>(src) + i) : make_int2(0, 0);
        w[2 * i] = (uint32_t)t.x;
        w[2 * i + 1] = (uint32_t)t.y;
      }
    }
    // scale 1/2: row pass two rows of the index set at a time (FP32x2), the
    // odd last row alone; only the set's columns are dequantized (the others
    // have an exactly-zero basis and are never read).  (At 1/4 the pairing
    // measured no gain: c3b 0.0370 vs 0.0371 ms, c5 +0.7 %; r02q.)
    constexpr int kRowStep = K == 2 ? 2 : 1;
#pragma unroll
    for (int i = 0; i < NS; i += kRowStep) {
      const int va = packed_set(K, i);
      const bool two = kRowStep == 2 && i + 1 < NS;
      const int vb = two ? packed_set(K, i + 1) : va;
      float da[8], db[8];
      if constexpr (PACKED) {
#pragma unroll
        for (int u = 0; u < 8; ++u) { da[u] = 0.f; db[u] = 0.f; }
#pragma unroll
        for (int jj = 0; jj < NS; ++jj) {
          da[packed_set(K, jj)] = half_of(w, i * NS + jj);
          if (two) db[packed_set(K, jj)] = half_of(w, (i + 1) * NS + jj);
        }
      } else {
        unpack_row(act ? __ldg(reinterpret_cast<const int4*>(src) + va) : make_int4(0, 0, 0, 0), da);
        if (two) unpack_row(act ? __ldg(reinterpret_cast<const int4*>(src) + vb) : make_int4(0, 0, 0, 0), db);
      }
      if (two) {
        float2 d[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) d[u] = make_float2(0.f, 0.f);
#pragma unroll
        for (int jj = 0; jj < NS; ++jj) {
          const int u = packed_set(K, jj);
          d[u] = __fmul2_rn(make_float2(da[u], db[u]), make_float2(q[va * 8 + u], q[vb * 8 + u]));
        }
        if (va == 0) d[0].x += 128.5f;      // level shift + rounding offset (DC weight is exactly 1)
        float2 o[P];
        if constexpr (K == 2) idct4x2(d, o); else idct2x2(d, o);
#pragma unroll
        for (int j = 0; j < P; ++j) { g[va][j] = o[j].x; g[vb][j] = o[j].y; }
      } else {
#pragma unroll
        for (int u = 0; u < 8; ++u) da[u] *= q[va * 8 + u];
        if (va == 0) da[0] += 128.5f;
        float o[P];
        if constexpr (K == 2) idct4(da, o); else idct2(da, o);
#pragma unroll
        for (int j = 0; j < P; ++j) g[va][j] = o[j];
      }
    }
#pragma unroll
    for (int x = 0; x < P; ++x) {
      float col[8], f[P];
#pragma unroll
      for (int v = 0; v < 8; ++v) col[v] = g[v][x];
      if constexpr (K == 2) idct4(col, f); else idct2(col, f);
#pragma unroll
      for (int y = 0; y < P; ++y) {
        const uint32_t b = floor_u8(f[y]);
        px[y][0] = (x == 0) ? b : (px[y][0] | (b << (8 * x)));
      }
    }
  }
}

// ------------------------------------------------------------- colour -----
// Reading R6.  R and B in fp32: t = c16 * k + (Y + c), floor+clamp in one
// F2I.U8.FLOOR.  Exactness: the fractional parts of the exact values are
// multiples of 1/8000 (R) and 1/4000 (B); the fp32 evaluation error is
// < 6.1e-5 and cB carries a +2^-13 bias so that B's two exact ties
// (Cb - 128 = +-125) round up; both bounds are verified exhaustively over all
// (Y, c16) by tests/test_color_fp32.py.  G = Y + floor((K1 - 43017 cb16 -
// 89267 cr16) / 2e6) - 136 in exact unsigned integers (K1 = 543917632).
__device__ __forceinline__ uint32_t colour(int Y, int cb16, int cr16) {
  const float yf = (float)Y;
  const uint32_t R = floor_u8(fmaf((float)cr16, c_basis.kR, yf + c_basis.cR));
  const uint32_t B = floor_u8(fmaf((float)cb16, c_basis.kB, yf + c_basis.cB));
  const uint32_t u = 543917632u - 43017u * (uint32_t)cb16 - 89267u * (uint32_t)cr16;
  const int G = min(max(Y + (int)(u / 2000000u) - 136, 0), 255);
  return R | ((uint32_t)G << 8) | (B << 16);
}

// Two pixels from 2^23-biased luma floats (one PRMT per sample builds the
// bits 0x4B0000YY = 2^23 + Y; subtracting 2^23 is exact), so no I2F is
// needed for Y; G uses the biased bits directly (the bias cancels in the
// IADD3).  Same IEEE fp32 operations as colour() otherwise.
__device__ __forceinline__ uint2 colour2m(uint32_t m0, uint32_t m1, int cb0, int cb1, int cr0, int cr1) {
  const float2 yf = __fadd2_rn(make_float2(__uint_as_float(m0), __uint_as_float(m1)), f2(-8388608.f));
  const float2 tr = __ffma2_rn(make_float2((float)cr0, (float)cr1), make_float2(c_basis.kR, c_basis.kR),
                               __fadd2_rn(yf, make_float2(c_basis.cR, c_basis.cR)));
  const float2 tb = __ffma2_rn(make_float2((float)cb0, (float)cb1), make_float2(c_basis.kB, c_basis.kB),
                               __fadd2_rn(yf, make_float2(c_basis.cB, c_basis.cB)));
  // constants from the constant bank (IMAD c[][] operand): as immediates the
  // compiler re-materialises them with a MOV per use under register pressure
  const uint32_t u0 = c_basis.gK1 + c_basis.gCb * (uint32_t)cb0 + c_basis.gCr * (uint32_t)cr0;
  const uint32_t u1 = c_basis.gK1 + c_basis.gCb * (uint32_t)cb1 + c_basis.gCr * (uint32_t)cr1;
  const uint32_t G0 = (uint32_t)min(max((int)(m0 + u0 / 2000000u - (0x4B000000u + 136u)), 0), 255);
  const uint32_t G1 = (uint32_t)min(max((int)(m1 + u1 / 2000000u - (0x4B000000u + 136u)), 0), 255);
  return make_uint2(__byte_perm(__byte_perm(floor_u8(tr.x), G0, 0x0040), floor_u8(tb.x), 0x5410),
                    __byte_perm(__byte_perm(floor_u8(tr.y), G1, 0x0040), floor_u8(tb.y), 0x5410));
}

__device__ __forceinline__ int ldu8(const uint8_t* p) { return *p; }

struct KParams {
  const DevRef* refs;              // per image: coefficient planes + kind
  const DevImage* kinds;           // per kind: geometry, strides, quant table ids
  const TileLayout* lays;          // per (kind, tile): the tile's layout (null: computed in the kernel)
  const int4* taps;                // tap regions referenced by TileLayout::tap_off
  int lay_stride;                  // layouts per kind
  const uint16_t* qtables;
  void* out;
  int OW, OH, tile_rows, tile_cols, n_col_tiles, n_row_tiles;
  int out_vec;                     // out is 16-B (fp32) / 8-B (fp16) aligned: vector stores allowed
  int rowrun;                      // > 0: output tasks walk runs of this many rows, reusing horizontal lerps (vertical magnification)
  const int4* cta_map;             // non-null: 1-D grid, CTA -> {image, oy0, oy1, 0}
  uint32_t magic;                  // 0x4B000000: bit pattern of 2^23 (byte -> float trick)
  float na[3], nb[3];              // y = x * na + nb = (x/255 - mean)/std
  int16_t* dbg_pl[3];              // debug planes (DEBUG instantiation only)
  int16_t* dbg_rgb;
  long long dbg_stride_y, dbg_stride_c, dbg_stride_rgb;
};

__device__ __forceinline__ uint32_t fdiv(uint32_t n, const FastDiv& f) {
  return f.d <= 1 ? n : __umulhi(n, f.m);
}

// byte b of x as float: PRMT (zero-extend) + I2FP (no XU-pipe I2F)
__device__ __forceinline__ float byte_f(uint32_t x, int b) {
  return __uint2float_rn(__byte_perm(x, 0u, 0x4440 + b));
}



template <int P>
__device__ __forceinline__ void put_row(uint8_t* d, const uint32_t (&w)[2]) {
  if constexpr (P == 8) *reinterpret_cast<uint2*>(d) = make_uint2(w[0], w[1]);
  else if constexpr (P == 4) *reinterpret_cast<uint32_t*>(d) = w[0];
  else if constexpr (P == 2) *reinterpret_cast<uint16_t*>(d) = (uint16_t)w[0];
  else *d = (uint8_t)w[0];
}


__device__ __forceinline__ uint32_t lds_u32(const uint8_t* p) { return *reinterpret_cast<const uint32_t*>(p); }

__device__ __forceinline__ uint32_t byte_of(const uint32_t (&w)[2], int e) {
  return ((e < 4 ? w[0] : w[1]) >> (8 * (e & 3))) & 255u;   // select: no dynamic register indexing
}

// Dynamic work distribution: lane 0 takes the next n tasks from a shared
// counter and broadcasts the base.
__device__ __forceinline__ int grab_chunk(int* ctr, int lane, int n = 32) {
  int chunk = 0;
  if (lane == 0) chunk = atomicAdd(ctr, n);
  return __shfl_sync(0xffffffffu, chunk, 0);
}

template <int K, bool F16, bool DEBUG, bool PACKED, int kThreads, int kYP, bool DB, bool GC, int CK>
__device__ __forceinline__ void smol_tile(const KParams& kp, const int n, const int oy0, const int oy1,
                                       const int ox0, const int ox1, const int lay_local) {
  constexpr int P = 8 / K;                 // decoded samples per block side
  constexpr int PC = 8 / CK;               // per chroma block side (= P unless chroma at twice the scale)
  static_assert(CK == K || GC, "chroma at another scale needs the generic-chroma rings");
  extern __shared__ __align__(16) uint8_t smem[];
  const int tid = threadIdx.x, lane = tid & 31;
  __shared__ DevImage im;
  __shared__ TileLayout L;
  __shared__ int ctr[2];                   // dynamic work counter of the output phase (ctr[1])
  // the image's descriptor (its kind, with the coefficient pointers of its
  // reference: the first 6 words of both) and the tile's layout, precomputed
  // by the host per (image kind, tile): copied in by all threads, a word each
  {
    static_assert(offsetof(DevImage, coef) == 0 && offsetof(DevRef, coef) == 0, "coef pointers lead both");
    static_assert(sizeof(DevImage) % 4 == 0 && sizeof(TileLayout) % 4 == 0, "word copies");
    const int kind = kp.refs[n].kind;
    const uint32_t* sr = reinterpret_cast<const uint32_t*>(kp.refs + n);
    const uint32_t* sk = reinterpret_cast<const uint32_t*>(kp.kinds + kind);
    uint32_t* di = reinterpret_cast<uint32_t*>(&im);
    for (int i = tid; i < (int)(sizeof(DevImage) / 4); i += kThreads) di[i] = i < 6 ? __ldg(sr + i) : __ldg(sk + i);
    if (kp.lays) {
      const uint32_t* sl = reinterpret_cast<const uint32_t*>(kp.lays + kind * kp.lay_stride + lay_local);
      uint32_t* dl = reinterpret_cast<uint32_t*>(&L);
      for (int i = tid; i < (int)(sizeof(TileLayout) / 4); i += kThreads) dl[i] = __ldg(sl + i);
    }
    if (tid == 0) ctr[1] = 0;
  }
  __syncthreads();
  if (!kp.lays) {                          // (uniform) the table did not fit: computed here
    if (tid == 0) tile_layout(im, K, oy0, oy1, ox0, ox1, L, kYP, GC);
    __syncthreads();
  }
  // chroma rings: 4:2:0 kernels (GC = false) keep 16 rows of half-width
  // chroma; generic-chroma kernels 32 rows of full width (4:2:2, 4:4:4)
  constexpr int kCP = c_pitch(kYP, GC);     // chroma ring pitch
  constexpr int kCR = c_ring(GC);           // chroma ring rows (power of 2)
  constexpr int kCS = c_slots(GC);          // + 2 guard slots
  const int cvs = GC ? im.vs : 2, chs = GC ? im.hs : 2;   // chroma subsampling factors
  float* qf = reinterpret_cast<float*>(smem + off_q(kYP, GC));
  int2* xt = reinterpret_cast<int2*>(smem + L.off_xt);
  int2* yt = reinterpret_cast<int2*>(smem + L.off_yt);
  uint8_t* yring = smem;
  uint8_t* cring = smem + off_c(kYP);
  uint32_t* rgb = reinterpret_cast<uint32_t*>(smem + off_rgb(kYP, GC));
  constexpr int kCStride = kCS * kCP;      // Cr ring follows the Cb ring
  const int ntw = ox1 - ox0, nth = oy1 - oy0;
  constexpr int rgb_p = rgb_pitch(kYP);     // RGB ring row pitch (u32), = L.rgb_p
  constexpr int pitch4 = rgb_p * 4;         // in bytes

  // ---- prologue: dequant tables (Q/8, exact) and bilinear taps ----------
  // Taps use exact-integer coordinates (R9).  Where the upper tap is clamped
  // (i1 == i0) its weight is zeroed so the kernel may always read i0 + 1.
  for (int i = tid; i < 3 * 64; i += kThreads) {
    int e = i & 63;
    qf[i] = (float)kp.qtables[im.qidx[i >> 6] * 64 + e] * 0.125f;
  }
  // x taps per output-pixel pair {byte offset of x0 (a), (b), w (a), w (b)},
  // so a pair's weights load into an adjacent register pair for FFMA2.
  // Output task q (pixels 4q .. 4q+3) reads pair A at [q] and pair B at
  // [nq4 + q]: consecutive lanes read consecutive 16-B entries.
  // y taps per output row: {byte offset of RGB ring row i0 | i1 << 16, w}
  // (row i0 + 1 is at +pitch4: the ring's guard slot mirrors slot 0).
  // Precomputed per (image kind, tile) by the host when it could (copied
  // in), else computed here (smol_geom.cuh tile_xtap / tile_ytap).
  const int nq4 = (ntw + 3) >> 2;
  if (L.tap_off >= 0) {
    const int4* src = kp.taps + L.tap_off;
    int4* dst = reinterpret_cast<int4*>(smem + L.off_xt);
    for (int i = tid; i < tile_tap_bytes(L) / 16; i += kThreads) dst[i] = src[i];
  } else {
    for (int i = tid; i < 4 * nq4; i += kThreads) tile_xtap(im, L, i, reinterpret_cast<int*>(xt));
    for (int i = tid; i < nth; i += kThreads) tile_ytap(im, L, i, pitch4, reinterpret_cast<int*>(yt));
  }
  if (im.gray)       // grayscale: neutral chroma everywhere in the rings (read only by colour)
    for (int i = tid; i < 2 * kCStride / 4; i += kThreads) reinterpret_cast<uint32_t*>(cring)[i] = 0x80808080u;
  const int nbx0 = L.bx1[0] - L.bx0[0] + 1, nbxc = L.bx1[1] - L.bx0[1] + 1;
  const FastDiv fd_y = L.fd_y, fd_c = L.fd_c;      // (divisors precomputed with the layout)
  const int ntask4 = L.rgb_w >> 2;          // 4-column colour tasks per quad row
  const FastDiv fd_t4 = L.fd_t4;
  const FastDiv fd_q4 = L.fd_q4;
  const bool vec4 = ((kp.OW & 3) == 0) && ((ox0 & 3) == 0) && kp.out_vec;
  const uint32_t plane_sz = (uint32_t)kp.OH * kp.OW;   // < 2^31 elements (host-checked)
  using OutT = typename std::conditional<F16, __half, float>::type;
  OutT* const outb = reinterpret_cast<OutT*>(kp.out) + ((size_t)n * 3 * kp.OH + oy0) * kp.OW + ox0;
  __syncthreads();

  // ---- IDCT of one rolling step's ROI blocks (static: thread per block) --
  auto idct_step = [&](int s) {
    const int R = L.r0 + kStepRows * s;
    const int yb0 = max(L.by0[0], R / P), yb1 = min(L.by1[0], (R + kStepRows) / P - 1);
    const int Rc = GC ? R / cvs : (R >> 1), crows = GC ? kStepRows / cvs : kStepRows / 2;  // chroma rows of the step
    const int cb0 = (s == 0) ? L.by0[1] : max(L.by0[1], Rc / PC);
    const int cb1 = min(L.by1[1], (Rc + crows) / PC - 1);
    const int ny = max(0, yb1 - yb0 + 1) * nbx0;
    const int nc = max(0, cb1 - cb0 + 1) * nbxc;
    const int ntask = ny + 2 * nc;
    // scale 1/8: one DC load per block; unrolled so several loads are in
    // flight per thread
#pragma unroll(K == 8 ? 4 : 1)
    for (int base = tid & ~31; base < ntask; base += kThreads) {
      const int t = base + lane;
      const bool act = t < ntask;
      int c = 0, brow = 0, bcol = 0;
      if (t < ny) {
        brow = (int)fdiv((uint32_t)t, fd_y);
        bcol = t - brow * nbx0;
        brow += yb0;
      } else if (act) {
        int tt = t - ny;
        c = 1 + (tt >= nc);
        tt -= (c - 1) * nc;
        brow = (int)fdiv((uint32_t)tt, fd_c);
        bcol = tt - brow * nbxc;
        brow += cb0;
      }
      const int16_t* src = im.coef[c] + (size_t)brow * im.stride[c] + (size_t)(L.bx0[c] + bcol) * BlockFmt<K, PACKED, DB>::kElems;
      uint32_t px[8][2];
      if constexpr (CK == K) {
        decode_block<K, PACKED, DB>(act, src, qf + c * 64, px);
      } else {
        // luma and chroma blocks decode at different scales: each variant
        // runs (warp-uniformly) for the warps holding such blocks
        const bool isy = c == 0;
        uint32_t pc[8][2];
        if (__any_sync(0xffffffffu, act && isy)) decode_block<K, PACKED, DB>(act && isy, src, qf + c * 64, px);
        if (__any_sync(0xffffffffu, act && !isy)) {
          decode_block<CK, PACKED, DB>(act && !isy, src, qf + c * 64, pc);
          if (!isy) {
#pragma unroll
            for (int y = 0; y < 8; ++y) { px[y][0] = pc[y][0]; px[y][1] = pc[y][1]; }
          }
        }
      }
      if (!act) continue;
      if (c == 0) {
        uint8_t* d = yring + bcol * P;
#pragma unroll
        for (int y = 0; y < P; ++y) put_row<P>(d + ((brow * P + y) & (kYRing - 1)) * kYP, px[y]);
      } else {
        uint8_t* d = cring + (c - 1) * kCStride + bcol * PC + kCPad;
        const int gx0 = (L.bx0[c] + bcol) * PC;
        const bool edge = (gx0 == 0) || (gx0 <= im.Wc - 1 && im.Wc - 1 < gx0 + PC);
#pragma unroll
        for (int y = 0; y < PC; ++y) {
          const int r = brow * PC + y;
          const int rs = r & (kCR - 1);
          // slot rs+1, plus the guard mirrors (slot 0 = kCR, slot kCR+1 = 1)
          for (int k = 0; k < 1 + (rs == kCR - 1 || rs == 0); ++k) {
            uint8_t* row = d + (k == 0 ? rs + 1 : (rs == kCR - 1 ? 0 : kCS - 1)) * kCP;
            put_row<PC>(row, px[y]);
            if (edge) {
              // replicate image-edge chroma columns into the neighbours the
              // triangle filter reads (reading R2: indices clamp at the edges)
              if (gx0 == 0) row[-1] = (uint8_t)byte_of(px[y], 0);
              const int e = im.Wc - 1 - gx0;
              if (e >= 0 && e < PC) row[e + 1] = (uint8_t)byte_of(px[y], e);
            }
          }
        }
      }
    }
  };

  // per-step schedule, computed once: ready_s = last RGB row available after
  // step s (monotone), done_s = output rows whose lower tap row is <= ready_s
  // (taps are monotone: binary search)
  int2* st = reinterpret_cast<int2*>(smem + L.off_st);
  for (int s = tid; s < L.nsteps; s += kThreads) {
    const int ready = max(L.ly0 - 1, ready_after(L, im.Hc, s, cvs));
    int lo = 0, hi = nth;
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if ((int)((uint32_t)yt[mid].x >> 16) <= ready) lo = mid + 1; else hi = mid;
    }
    st[s] = make_int2(ready, lo);
  }
  int ready_prev = L.ly0 - 1;
  int done_prev = 0;                       // output rows of the tile finished
  idct_step(0);
  __syncthreads();

  for (int s = 0; s < L.nsteps; ++s) {
    const int2 sts = st[s];
    const int ready = sts.x;
    if (tid == 0) ctr[1] = 0;

    if constexpr (DEBUG) {
      // decoded samples of this step's block rows, clipped to the footprint
      const int R = L.r0 + kStepRows * s;
      for (int c = 0; c < 3; ++c) {
        const int W = c ? im.Wc : im.Wd, Hh = c ? im.Hc : im.Hd;
        int rlo, rhi;
        if (c == 0) { rlo = max(max(L.by0[0], R / P) * P, L.ly0); rhi = min(min(L.by1[0], (R + kStepRows) / P - 1) * P + P - 1, L.ly1); }
        else {
          const int Rc = R / cvs;
          rlo = max(((s == 0) ? L.by0[1] : max(L.by0[1], Rc / PC)) * PC, L.cy0);
          rhi = min(min(L.by1[1], (Rc + kStepRows / cvs) / PC - 1) * PC + PC - 1, L.cy1);
        }
        const int x0 = c ? L.cx0 : L.lx0, x1 = c ? L.cx1 : L.lx1;
        int16_t* dst = kp.dbg_pl[c] + n * (c ? kp.dbg_stride_c : kp.dbg_stride_y);
        for (int y = rlo; y <= rhi; ++y)
          for (int x = x0 + tid; x <= x1; x += kThreads)
            if (y < Hh && x < W)
              dst[(size_t)y * W + x] = c == 0 ? yring[(y & (kYRing - 1)) * kYP + (x - L.xbase[0])]
                                              : cring[(c - 1) * kCStride + ((y & (kCR - 1)) + 1) * kCP +
                                                      (x - L.xbase[c] + kCPad)];
      }
    }

    // ---- prefetch step s+1's ROI block rows into L2 (TMA bulk prefetch) --
    // one contiguous segment per (component, block row); the IDCT of step
    // s+1 (next phase) then hits L2 instead of waiting on HBM.
    // (not for dense blocks at scale 1/8: only the DC's 32-B sector is read
    // there, and a row prefetch would pull all 128 B of every block)
    if ((K != 8 || PACKED) && s + 1 < L.nsteps && tid >= kThreads - 32) {
      const int R = L.r0 + kStepRows * (s + 1);
      const int yb0 = max(L.by0[0], R / P), yb1 = min(L.by1[0], (R + kStepRows) / P - 1);
      const int Rc = GC ? R / cvs : (R >> 1), crows = GC ? kStepRows / cvs : kStepRows / 2;
      const int cb0 = max(L.by0[1], Rc / PC);
      const int cb1 = min(L.by1[1], (Rc + crows) / PC - 1);
      const int ny = max(0, yb1 - yb0 + 1), nc = max(0, cb1 - cb0 + 1);
      for (int k = lane; k < ny + 2 * nc; k += 32) {
        int c = 0, brow = yb0 + k;
        if (k >= ny) { c = 1 + (k - ny >= nc); brow = cb0 + (k - ny) - (c - 1) * nc; }
        // 16-B aligned segment [bx0 * S, (bx1 + 1) * S) of the (16-B padded) block row
        constexpr int SB = BlockFmt<K, PACKED, DB>::kElems * 2;
        const uint32_t lo = ((uint32_t)L.bx0[c] * SB) & ~15u, hi = ((uint32_t)(L.bx1[c] + 1) * SB + 15u) & ~15u;
        const char* p = reinterpret_cast<const char*>(im.coef[c] + (size_t)brow * im.stride[c]) + lo;
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" :: "l"(p), "r"(hi - lo) : "memory");
      }
    }


    // ---- upsample + colour of the RGB rows that became ready -------------
    // A task is 2x4 luma pixels (rows 2j, 2j+1; cols 2i .. 2i+3) sharing a
    // 3x4 chroma neighbourhood.  Steps end on odd rows (ready_after), so
    // quads never straddle steps; at the footprint's first/last row a quad
    // may include one row outside it (computed, never read).
    if constexpr (GC) {
      // generic chroma (4:2:2, 4:4:4; reading R2 per axis): along a
      // subsampled axis the triangle 3/4, 1/4, along an unsubsampled one the
      // sample itself (weight 4/4); values in 1/16 units as for 4:2:0
      const int j0 = (ready_prev + 1) >> 1;
      const int nq = ready > ready_prev ? (ready >> 1) - j0 + 1 : 0;
      const int ntaskc = nq * ntask4;
      for (int t = tid; t < ntaskc; t += kThreads) {
        const int rr = (int)fdiv((uint32_t)t, fd_t4);
        const int p = t - rr * ntask4;
        const int j = j0 + rr;                               // luma rows 2j, 2j+1
        const int lx = L.rgb_x0 + 4 * p;                     // luma column of the quad
        const int cc = (chs == 2 ? lx >> 1 : lx) - L.xbase[1] + kCPad;   // ring column of its chroma
        int cbq[8], crq[8];
#pragma unroll
        for (int comp = 0; comp < 2; ++comp) {
          const uint8_t* base = cring + comp * kCStride + cc;
          auto hrow = [&](int crow, int (&h)[4]) {           // horizontal filter of chroma row crow
            const uint8_t* r = base + ((crow & (kCR - 1)) + 1) * kCP;
            if (chs == 2) {
              const int a = ldu8(r - 1), m = ldu8(r), n2 = ldu8(r + 1), z = ldu8(r + 2);
              h[0] = 3 * m + a; h[1] = 3 * m + n2; h[2] = 3 * n2 + m; h[3] = 3 * n2 + z;
            } else {
#pragma unroll
              for (int x = 0; x < 4; ++x) h[x] = 4 * ldu8(r + x);
            }
          };
          int* qv = comp ? crq : cbq;
          if (cvs == 2) {
            int h0[4], h1[4], h2[4];
            hrow(j > 0 ? j - 1 : 0, h0);
            hrow(j, h1);
            hrow(j < im.Hc - 1 ? j + 1 : j, h2);
#pragma unroll
            for (int x = 0; x < 4; ++x) { qv[x] = 3 * h1[x] + h0[x]; qv[4 + x] = 3 * h1[x] + h2[x]; }
          } else {
            int ha[4], hb[4];
            hrow(min(2 * j, im.Hc - 1), ha);
            hrow(min(2 * j + 1, im.Hc - 1), hb);
#pragma unroll
            for (int x = 0; x < 4; ++x) { qv[x] = 4 * ha[x]; qv[4 + x] = 4 * hb[x]; }
          }
        }
        const uint8_t* yr = yring + ((2 * j) & (kYRing - 1)) * kYP + (lx - L.xbase[0]);
        const uint32_t y0 = *reinterpret_cast<const uint32_t*>(yr);
        const uint32_t y1 = *reinterpret_cast<const uint32_t*>(yr + kYP);
        const int slot = rgb_slot(2 * j);
        uint32_t* r0p = rgb + slot * rgb_p + (lx - L.rgb_x0);
        const uint32_t mg = 0x4B000000u;
        const uint2 t01 = colour2m(__byte_perm(y0, mg, 0x7540), __byte_perm(y0, mg, 0x7541), cbq[0], cbq[1], crq[0], crq[1]);
        const uint2 t23 = colour2m(__byte_perm(y0, mg, 0x7542), __byte_perm(y0, mg, 0x7543), cbq[2], cbq[3], crq[2], crq[3]);
        const uint2 b01 = colour2m(__byte_perm(y1, mg, 0x7540), __byte_perm(y1, mg, 0x7541), cbq[4], cbq[5], crq[4], crq[5]);
        const uint2 b23 = colour2m(__byte_perm(y1, mg, 0x7542), __byte_perm(y1, mg, 0x7543), cbq[6], cbq[7], crq[6], crq[7]);
        const uint4 top = make_uint4(t01.x, t01.y, t23.x, t23.y);
        *reinterpret_cast<uint4*>(r0p) = top;
        *reinterpret_cast<uint4*>(r0p + rgb_p) = make_uint4(b01.x, b01.y, b23.x, b23.y);
        if (slot == 0) *reinterpret_cast<uint4*>(r0p + kRgbRing * rgb_p) = top;   // guard row
      }
    } else
    {
      const int j0 = (ready_prev + 1) >> 1;
      const int nq = ready > ready_prev ? (ready >> 1) - j0 + 1 : 0;
      const int ntaskc = nq * ntask4;
      // colour tasks all cost the same and nothing else runs in this phase:
      // a static round-robin needs no work counter (running the partial last
      // round as half tasks, or unrolling two tasks per thread, measured
      // slower, r02)
      for (int t = tid; t < ntaskc; t += kThreads) {
        const int rr = (int)fdiv((uint32_t)t, fd_t4);
        const int p = t - rr * ntask4;
        const int j = j0 + rr;                               // chroma row of the quads
        const int i = (L.rgb_x0 >> 1) + 2 * p;               // chroma column of the left quad
        const uint8_t* c1 = cring + ((j & (kCR - 1)) + 1) * kCP + (i - L.xbase[1] + kCPad);
        const uint8_t* c0 = c1 + (j > 0 ? -kCP : 0);               // row j-1 (clamped at the top)
        const uint8_t* c2 = c1 + (j < im.Hc - 1 ? kCP : 0);        // row j+1 (clamped at the bottom)
        int cbq[8], crq[8];                                  // [row 0: 4 cols][row 1: 4 cols]
#pragma unroll
        for (int comp = 0; comp < 2; ++comp) {
          const int o = comp * kCStride;
          int h[3][4];                                       // horizontal 3/1 taps per chroma row
          const uint8_t* rows[3] = {c0, c1, c2};
#pragma unroll
          for (int r = 0; r < 3; ++r) {
            const int a = ldu8(rows[r] + o - 1), m = ldu8(rows[r] + o), n2 = ldu8(rows[r] + o + 1),
                      z = ldu8(rows[r] + o + 2);
            h[r][0] = 3 * m + a;     // col 2i
            h[r][1] = 3 * m + n2;    // col 2i+1
            h[r][2] = 3 * n2 + m;    // col 2i+2
            h[r][3] = 3 * n2 + z;    // col 2i+3
          }
          int* qv = comp ? crq : cbq;
#pragma unroll
          for (int x = 0; x < 4; ++x) {
            qv[x] = 3 * h[1][x] + h[0][x];       // row 2j
            qv[4 + x] = 3 * h[1][x] + h[2][x];   // row 2j+1
          }
        }
        const uint8_t* yr = yring + ((2 * j) & (kYRing - 1)) * kYP + (2 * i - L.xbase[0]);
        const uint32_t y0 = *reinterpret_cast<const uint32_t*>(yr);
        const uint32_t y1 = *reinterpret_cast<const uint32_t*>(yr + kYP);
        const int slot = rgb_slot(2 * j);
        uint32_t* r0p = rgb + slot * rgb_p + (2 * i - L.rgb_x0);
        const uint32_t mg = 0x4B000000u;
        const uint2 t01 = colour2m(__byte_perm(y0, mg, 0x7540), __byte_perm(y0, mg, 0x7541), cbq[0], cbq[1], crq[0], crq[1]);
        const uint2 t23 = colour2m(__byte_perm(y0, mg, 0x7542), __byte_perm(y0, mg, 0x7543), cbq[2], cbq[3], crq[2], crq[3]);
        const uint2 b01 = colour2m(__byte_perm(y1, mg, 0x7540), __byte_perm(y1, mg, 0x7541), cbq[4], cbq[5], crq[4], crq[5]);
        const uint2 b23 = colour2m(__byte_perm(y1, mg, 0x7542), __byte_perm(y1, mg, 0x7543), cbq[6], cbq[7], crq[6], crq[7]);
        const uint4 top = make_uint4(t01.x, t01.y, t23.x, t23.y);
        *reinterpret_cast<uint4*>(r0p) = top;
        *reinterpret_cast<uint4*>(r0p + rgb_p) = make_uint4(b01.x, b01.y, b23.x, b23.y);
        if (slot == 0) *reinterpret_cast<uint4*>(r0p + kRgbRing * rgb_p) = top;   // guard row
      }
    }
    __syncthreads();

    if constexpr (DEBUG) {
      int16_t* dst = kp.dbg_rgb + n * kp.dbg_stride_rgb;
      for (int y = ready_prev + 1; y <= ready; ++y)
        for (int x = L.lx0 + tid; x <= L.lx1; x += kThreads) {
          const uint32_t v = rgb[rgb_slot(y) * rgb_p + (x - L.rgb_x0)];
          const size_t o = ((size_t)y * im.Wd + x) * 3;
          dst[o] = v & 255; dst[o + 1] = (v >> 8) & 255; dst[o + 2] = (v >> 16) & 255;
        }
    }

    const int done = sts.y;

    // ---- next step's IDCT (writes only Y/chroma rings: no reader now) ----
    if (s + 1 < L.nsteps) idct_step(s + 1);

    if (K != 1 && kp.rowrun)      // (scale 1: measured no gain at c2; keeps the K=1 kernel's registers)
    // ---- bilinear + normalize + NCHW store: a task is one 4-pixel column
    // quad over a run of up to kRun consecutive output rows.  Walking down
    // the run, the horizontal lerps of a source row are reused while the
    // row's taps do not move: the same (i0, i0+1) pair keeps both, a pair
    // one row lower keeps the old bottom lerp as the new top.  Bit-identical
    // to recomputing them (same operations on the same samples).
    {
      const int kRun = kp.rowrun;        // rows per run (host: longer under stronger magnification)
      const int nrows = done - done_prev;
      const int ngr = (nrows + kRun - 1) / kRun;
      const int ntasko = ngr * nq4;
      const float2 na0 = f2(kp.na[0]), na1 = f2(kp.na[1]), na2 = f2(kp.na[2]);
      const float2 nb0 = f2(kp.nb[0]), nb1 = f2(kp.nb[1]), nb2 = f2(kp.nb[2]);
      const uint32_t magic = kp.magic;     // 0x4B000000 (2^23), kept in a register
      constexpr bool kOutStatic = SMOL_OUT_STATIC == 1 || (SMOL_OUT_STATIC == 2 && K != 1);
      for (int chunk = kOutStatic ? (tid >> 5) * 32 : 0;; chunk += kThreads) {
        if constexpr (!kOutStatic) {
          if (ctr[1] >= ntasko) break;           // (no atomic once the phase's tasks are gone)
          chunk = grab_chunk(&ctr[1], lane, 32);
        }
        if (chunk >= ntasko) break;
        const int t = chunk + lane;
        if (t >= ntasko) continue;
        const int gi = (int)fdiv((uint32_t)t, fd_q4);
        const int q = t - gi * nq4;
        const int ra = done_prev + gi * kRun, rb = min(ra + kRun, done);
        const int ox = 4 * q;
        const int4* xt4 = reinterpret_cast<const int4*>(xt);
        const int4 txa = xt4[q];          // taps of ox, ox+1
        const int4 txb = xt4[nq4 + q];    // taps of ox+2, ox+3 (padded)
        const float2 wxa = make_float2(__int_as_float(txa.z), __int_as_float(txa.w));
        const float2 wxb = make_float2(__int_as_float(txb.z), __int_as_float(txb.w));
        const bool vst = vec4 && ox + 4 <= ntw;
        float2 T[3][2], B[3][2];          // horizontal lerps of the top / bottom source rows [ch][pixel pair]
        // horizontal lerps of one RGB ring row (byte offset ro) for the quad
        auto hlerp = [&](int ro, float2 (&H)[3][2]) {
          const uint8_t* row = reinterpret_cast<const uint8_t*>(rgb) + ro;
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int4 tx = e == 0 ? txa : txb;
            const float2 wx = e == 0 ? wxa : wxb;
            const uint32_t p0 = lds_u32(row + tx.x), p1 = lds_u32(row + tx.x + 4);
            const uint32_t q0 = lds_u32(row + tx.y), q1 = lds_u32(row + tx.y + 4);
#pragma unroll
            for (int ch = 0; ch < 3; ++ch) {
              const int sel = 0x7540 + ch;
              // bytes become 2^23 + b floats by one PRMT (exact), the bias cancels in b - a
              const float2 fa = make_float2(__uint_as_float(__byte_perm(p0, magic, sel)), __uint_as_float(__byte_perm(q0, magic, sel)));
              const float2 fb = make_float2(__uint_as_float(__byte_perm(p1, magic, sel)), __uint_as_float(__byte_perm(q1, magic, sel)));
              H[ch][e] = __ffma2_rn(wx, __ffma2_rn(fa, f2(-1.f), fb), __fadd2_rn(fa, f2(-8388608.f)));
            }
          }
        };
        int cur = -1;                     // ring byte offset of the current top row
        // output pointer walks down the run (one 64-bit add per row instead of
        // re-deriving the task's column per row)
        OutT* ot = outb + (uint32_t)(ra * kp.OW + ox);
#pragma unroll 1
        for (int r = ra; r < rb; ++r, ot += kp.OW) {
          const int2 ty = yt[r];
          const int ro = ty.x & 0xffff;
          if (ro != cur) {
            if (ro == cur + pitch4) {     // one row down: old bottom becomes the top
#pragma unroll
              for (int ch = 0; ch < 3; ++ch) { T[ch][0] = B[ch][0]; T[ch][1] = B[ch][1]; }
            } else {
              hlerp(ro, T);
            }
            hlerp(ro + pitch4, B);
            cur = ro;
          }
          const float2 wy2 = f2(__int_as_float(ty.y));
          float y[3][4];
#pragma unroll
          for (int ch = 0; ch < 3; ++ch)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
              const float2 v = __ffma2_rn(wy2, __ffma2_rn(T[ch][e], f2(-1.f), B[ch][e]), T[ch][e]);
              const float2 yn = __ffma2_rn(v, ch == 0 ? na0 : ch == 1 ? na1 : na2, ch == 0 ? nb0 : ch == 1 ? nb1 : nb2);
              y[ch][2 * e] = yn.x;
              y[ch][2 * e + 1] = yn.y;
            }
          if (vst) {
#pragma unroll
            for (int ch = 0; ch < 3; ++ch) {
              if constexpr (F16) {
                const __half2 h0 = __floats2half2_rn(y[ch][0], y[ch][1]);
                const __half2 h1 = __floats2half2_rn(y[ch][2], y[ch][3]);
                uint2 v;
                v.x = *reinterpret_cast<const uint32_t*>(&h0);
                v.y = *reinterpret_cast<const uint32_t*>(&h1);
                __stcs(reinterpret_cast<uint2*>(ot + ch * plane_sz), v);
              } else {
                __stcs(reinterpret_cast<float4*>(ot + ch * plane_sz),
                       make_float4(y[ch][0], y[ch][1], y[ch][2], y[ch][3]));
              }
            }
          } else {
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              if (ox + e >= ntw) break;
#pragma unroll
              for (int ch = 0; ch < 3; ++ch) {
                if constexpr (F16) ot[e + ch * plane_sz] = __float2half_rn(y[ch][e]);
                else ot[e + ch * plane_sz] = y[ch][e];
              }
            }
          }
        }
      }
    }
    else
    // ---- bilinear + normalize + NCHW store, 4 output pixels per task -----
    {
      const int ntasko = (done - done_prev) * nq4;
      const float2 na0 = f2(kp.na[0]), na1 = f2(kp.na[1]), na2 = f2(kp.na[2]);
      const float2 nb0 = f2(kp.nb[0]), nb1 = f2(kp.nb[1]), nb2 = f2(kp.nb[2]);
      const uint32_t magic = kp.magic;     // 0x4B000000 (2^23), kept in a register
      // dynamic warp-chunk grabbing balances output tasks against the IDCT of
      // step s+1 running in the same phase; SMOL_OUT_STATIC (1: always, 2:
      // reduced scales only, where that IDCT is small) strides statically
      constexpr bool kOutStatic = SMOL_OUT_STATIC == 1 || (SMOL_OUT_STATIC == 2 && K != 1);
      constexpr int kPer = kOutStatic ? 1 : SMOL_OUT_PER_GRAB;   // tasks per lane per grab (unrolled)
      for (int chunk = kOutStatic ? (tid >> 5) * 32 : 0;; chunk += kThreads * kPer) {
        if constexpr (!kOutStatic) chunk = grab_chunk(&ctr[1], lane, 32 * kPer);
        if (chunk >= ntasko) break;
#pragma unroll
       for (int h = 0; h < kPer; ++h) {
        const int t0 = chunk + 32 * h + lane;
        // (predicated, no break, so the compiler can interleave unrolled tasks)
        const bool live = t0 < ntasko;
        if (kPer == 1 && !live) break;
        const int t = live ? t0 : ntasko - 1;
        const int rr = (int)fdiv((uint32_t)t, fd_q4);
        const int r = done_prev + rr;
        const int ox = 4 * (t - rr * nq4);
        const int2 ty = yt[r];
        const float wy = __int_as_float(ty.y);
        const uint8_t* row0 = reinterpret_cast<const uint8_t*>(rgb) + (ty.x & 0xffff);
        const uint8_t* row1 = row0 + pitch4;
        float y[3][4];
        const int4* xt4 = reinterpret_cast<const int4*>(xt);
        const int4 txa = xt4[ox >> 2];          // taps of ox, ox+1
        const int4 txb = xt4[nq4 + (ox >> 2)];  // taps of ox+2, ox+3 (padded)
        const float2 wy2 = f2(wy);
#pragma unroll
        for (int e = 0; e < 4; e += 2) {
          // two output pixels per packed FP32x2 instruction; bytes become
          // 2^23 + b floats by one PRMT (exact), the bias cancels in b - a
          const int4 tx = e == 0 ? txa : txb;
          const float2 wx = make_float2(__int_as_float(tx.z), __int_as_float(tx.w));
          const uint32_t p00 = lds_u32(row0 + tx.x), p01 = lds_u32(row0 + tx.x + 4);
          const uint32_t p10 = lds_u32(row1 + tx.x), p11 = lds_u32(row1 + tx.x + 4);
          const uint32_t q00 = lds_u32(row0 + tx.y), q01 = lds_u32(row0 + tx.y + 4);
          const uint32_t q10 = lds_u32(row1 + tx.y), q11 = lds_u32(row1 + tx.y + 4);
#pragma unroll
          for (int ch = 0; ch < 3; ++ch) {
            const int sel = 0x7540 + ch;
            const float2 fa = make_float2(__uint_as_float(__byte_perm(p00, magic, sel)), __uint_as_float(__byte_perm(q00, magic, sel)));
            const float2 fb = make_float2(__uint_as_float(__byte_perm(p01, magic, sel)), __uint_as_float(__byte_perm(q01, magic, sel)));
            const float2 fc = make_float2(__uint_as_float(__byte_perm(p10, magic, sel)), __uint_as_float(__byte_perm(q10, magic, sel)));
            const float2 fd = make_float2(__uint_as_float(__byte_perm(p11, magic, sel)), __uint_as_float(__byte_perm(q11, magic, sel)));
            const float2 tp = __ffma2_rn(wx, __ffma2_rn(fa, f2(-1.f), fb), __fadd2_rn(fa, f2(-8388608.f)));
            const float2 bt = __ffma2_rn(wx, __ffma2_rn(fc, f2(-1.f), fd), __fadd2_rn(fc, f2(-8388608.f)));
            const float2 v = __ffma2_rn(wy2, __ffma2_rn(tp, f2(-1.f), bt), tp);
            const float2 yn = __ffma2_rn(v, ch == 0 ? na0 : ch == 1 ? na1 : na2, ch == 0 ? nb0 : ch == 1 ? nb1 : nb2);
            y[ch][e] = yn.x;
            y[ch][e + 1] = yn.y;
          }
        }
        OutT* const ot = outb + (uint32_t)(r * kp.OW + ox);
        if (!live) {
        } else if (vec4 && ox + 4 <= ntw) {
#pragma unroll
          for (int ch = 0; ch < 3; ++ch) {
            if constexpr (F16) {
              const __half2 h0 = __floats2half2_rn(y[ch][0], y[ch][1]);
              const __half2 h1 = __floats2half2_rn(y[ch][2], y[ch][3]);
              uint2 v;
              v.x = *reinterpret_cast<const uint32_t*>(&h0);
              v.y = *reinterpret_cast<const uint32_t*>(&h1);
              __stcs(reinterpret_cast<uint2*>(ot + ch * plane_sz), v);
            } else {
              __stcs(reinterpret_cast<float4*>(ot + ch * plane_sz),
                     make_float4(y[ch][0], y[ch][1], y[ch][2], y[ch][3]));
            }
          }
        } else {
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            if (ox + e >= ntw) break;
#pragma unroll
            for (int ch = 0; ch < 3; ++ch) {
              if constexpr (F16) ot[e + ch * plane_sz] = __float2half_rn(y[ch][e]);
              else ot[e + ch * plane_sz] = y[ch][e];
            }
          }
        }
       }
      }
    }
    __syncthreads();
    ready_prev = ready;
    done_prev = done;
  }
}

// Resident CTAs per SM the kernel is register-budgeted for: 24 warps at <= 80
// registers, except the tiny configuration at scales 1/2 and 1/4, whose IDCT
// fits 64 registers without spills: 8 CTAs (32 warps) per SM there for the
// latency-bound small footprints (c3b +5 %).  At 1/8 (DC only) the same
// change measured -11 % on c4 (profiles/r01p_occupancy.md), so it keeps 6.
template <int K>
__host__ __device__ constexpr int kCtasPerSm(int threads) {
  return ((K == 2 || K == 4) && threads == kThreadsTiny) ? 8 : 768 / threads;
}

// The fused kernel: one (image, row band, column band) tile per CTA.
// DB: Definition B reduced-scale IDCT (K = 2, 4 only; equal to A at 1, 1/8).
// CK: decode scale of the chroma blocks: K, or K/2 for libjpeg-turbo-style
// scaled decoding of 4:2:0 (chroma IDCT at twice the luma scale, no
// upsampling; reading R18; generic-chroma kernels only).
template <int K, bool F16, bool DEBUG, bool PACKED, int kThreads, int kYP, bool DB = false, bool GC = false,
          int CK = K>
__global__ void __launch_bounds__(kThreads, kCtasPerSm<K>(kThreads))
smol_fused_kernel(const __grid_constant__ KParams kp) {
  int n, oy0, oy1, ox0, ox1, local;
  if (kp.cta_map) {            // 1-D grid: per-CTA {image, oy0, oy1, layout} (full-width tiles)
    const int4 m = kp.cta_map[blockIdx.x];
    n = m.x; oy0 = m.y; oy1 = m.z; ox0 = 0; ox1 = kp.OW; local = m.w;
  } else {                     // 1-D grid: image-major, then row tile, then column tile
    const int per_img = kp.n_row_tiles * kp.n_col_tiles;
    n = blockIdx.x / per_img;
    local = blockIdx.x - n * per_img;
    const int trow = local / kp.n_col_tiles, tcol = local - trow * kp.n_col_tiles;
    oy0 = trow * kp.tile_rows; oy1 = min(kp.OH, oy0 + kp.tile_rows);
    ox0 = tcol * kp.tile_cols; ox1 = min(kp.OW, ox0 + kp.tile_cols);
  }
  smol_tile<K, F16, DEBUG, PACKED, kThreads, kYP, DB, GC, CK>(kp, n, oy0, oy1, ox0, ox1, local);
}

}  // namespace smol
