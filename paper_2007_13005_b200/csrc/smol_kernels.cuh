// smol_kernels.cuh -- the fused sm_100a kernel of the Smol preprocessing hot
// path: dequantize -> scaled IDCT -> u8 -> 4:2:0 upsample -> YCbCr->RGB ->
// bilinear resize + crop -> normalize -> NCHW, one CTA per (image, tile of
// output rows).  Decoded pixels live only in shared memory.
//
// Per CTA (256 threads):
//   stage 0  tile geometry, dequant table (Q/8 in fp32), per-column and
//            per-row bilinear taps (exact-integer coordinates, R9)
//   stage 1  every ROI block of the tile (Y, Cb, Cr): 8 lanes per block, lane
//            = coefficient row; one 128-bit load per lane (a warp reads 4
//            consecutive blocks = 512 contiguous bytes); row pass in
//            registers; transpose through smem; column pass; round/clamp to
//            u8 with one F2I.U8.FLOOR (reading R3) into the u8 planes
//   stage 2  upsample + colour for every footprint pixel -> packed RGBx u32
//   stage 3  bilinear + normalize per output pixel, coalesced NCHW stores
#pragma once
#include <cuda_fp16.h>
#include <stdint.h>

#include "smol_geom.cuh"

namespace smol {

// Basis constants, computed on the host in double from their definitions
// (smol_preproc.cu: init_basis) and uploaded once per device.
//   t[u][x]  = sqrt2 C(u) cos((2x+1) u pi/16), x < 4   (t[0][x] = 1, t[4][x] = +-1 exactly)
//   a2[j][u] = 1/2 sum_{x=2j}^{2j+1} t[u][x], j < 2    (a2[j][0] = 1, a2[j][4] = 0 exactly)
//   a4[u]    = 1/4 sum_{x=0}^{3} t[u][x]               (a4[0] = 1; 0 for u = 2, 4, 6)
// Output j and P-1-j are mirror images: t[u][7-x] = (-1)^u t[u][x] (same for a_k).
struct Basis {
  float t[8][4];
  float a2[2][8];
  float a4[8];
};

__constant__ Basis c_basis;

// 1-D transforms (reading R1, Definition A; separable form of the oracle's
// sum).  in[u], u = 0..7  ->  out[j], j = 0..P-1.  The FMA chains start from
// in[0] (weight exactly 1) and the exact +-1 / 0 entries so that DC-only and
// {0,4}-only inputs are transformed exactly.
template <int K> struct Idct1D;

template <> struct Idct1D<1> {
  static __device__ __forceinline__ void run(const float (&d)[8], float (&o)[8]) {
#pragma unroll
    for (int x = 0; x < 4; ++x) {
      float e = fmaf(d[4], c_basis.t[4][x], d[0]);
      e = fmaf(d[2], c_basis.t[2][x], e);
      e = fmaf(d[6], c_basis.t[6][x], e);
      float od = d[1] * c_basis.t[1][x];
      od = fmaf(d[3], c_basis.t[3][x], od);
      od = fmaf(d[5], c_basis.t[5][x], od);
      od = fmaf(d[7], c_basis.t[7][x], od);
      o[x] = e + od;
      o[7 - x] = e - od;
    }
  }
};

template <> struct Idct1D<2> {
  static __device__ __forceinline__ void run(const float (&d)[8], float (&o)[4]) {
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
};

template <> struct Idct1D<4> {
  static __device__ __forceinline__ void run(const float (&d)[8], float (&o)[2]) {
    float od = d[1] * c_basis.a4[1];
    od = fmaf(d[3], c_basis.a4[3], od);
    od = fmaf(d[5], c_basis.a4[5], od);
    od = fmaf(d[7], c_basis.a4[7], od);
    o[0] = d[0] + od;
    o[1] = d[0] - od;
  }
};

// Reading R3: clamp(floor(v + 128 + 1/2), 0, 255) in one F2I.U8.FLOOR (cvt
// saturates to the u8 range).
__device__ __forceinline__ uint32_t round_u8(float v) {
  uint32_t r;
  asm("cvt.rmi.sat.u8.f32 %0, %1;" : "=r"(r) : "f"(v + 128.5f));
  return r;
}

struct KParams {
  const DevImage* imgs;
  const uint16_t* qtables;
  void* out;
  int OW, OH, tile_rows;
  float na[3], nb[3];              // y = x * na + nb = (x/255 - mean)/std
  int16_t* dbg_pl[3];              // debug planes (DEBUG instantiation only)
  int16_t* dbg_rgb;
  long long dbg_stride_y, dbg_stride_c, dbg_stride_rgb;
};

// Reading R6, exact JFIF in integers: with chroma c16 in 1/16 units and
// d = c16 - 2048,  R = Y + floor((175250 dR + 10^6) / (2*10^6)),
// G = Y + floor((-43017 dB - 89267 dR + 10^6) / (2*10^6)),
// B = Y + floor((221500 dB + 10^6) / (2*10^6))   (1.402/16 = 175250/2e6 ...).
// floor division of a possibly negative numerator via an unsigned bias of
// 256 * 2e6 (all numerators stay below 2^31).
__device__ __forceinline__ int jfif_offset(int num) {
  return (int)((uint32_t)(num + 1000000 + 512000000) / 2000000u) - 256;
}
__device__ __forceinline__ uint32_t clamp255(int x) { return (uint32_t)min(max(x, 0), 255); }

template <int K, bool F16, bool DEBUG>
__global__ void __launch_bounds__(kThreads, 2)
smol_fused_kernel(const KParams kp) {
  constexpr int P = 8 / K;                 // decoded samples per block side
  extern __shared__ __align__(16) uint8_t smem[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int n = blockIdx.y;
  const int oy0 = blockIdx.x * kp.tile_rows;
  const int oy1 = min(kp.OH, oy0 + kp.tile_rows);
  const int OW = kp.OW;

  // Descriptor and tile geometry live in shared memory: per-component fields
  // are indexed with a runtime component id (no local-memory arrays).
  __shared__ DevImage im;
  __shared__ TileLayout L;
  if (tid == 0) {
    im = kp.imgs[n];
    tile_layout(im, K, OW, oy0, oy1, L);
  }
  __syncthreads();
  float* qf = reinterpret_cast<float*>(smem + L.off_q);
  int2* xt = reinterpret_cast<int2*>(smem + L.off_xt);
  int2* yt = reinterpret_cast<int2*>(smem + L.off_yt);
  uint32_t* rgb = reinterpret_cast<uint32_t*>(smem + L.off_rgb);
  float* scratch = reinterpret_cast<float*>(smem + L.off_rgb);   // aliases rgb (stage 1 only)

  // ---- stage 0: dequant table and taps ----------------------------------
  for (int i = tid; i < 3 * 64; i += kThreads) {
    const int c = i >> 6;
    qf[i] = (float)kp.qtables[im.qidx[c] * 64 + (i & 63)] * 0.125f;   // Q/8 (exact)
  }
  for (int ox = tid; ox < OW; ox += kThreads) {
    int i0, i1; float w;
    src_tap(im.left + ox, im.Wd, im.Wr, i0, i1, w);
    xt[ox] = make_int2((i0 - L.lx0) | ((i1 - L.lx0) << 16), __float_as_int(w));
  }
  for (int r = tid; r < oy1 - oy0; r += kThreads) {
    int i0, i1; float w;
    src_tap(im.top + oy0 + r, im.Hd, im.Hr, i0, i1, w);
    yt[r] = make_int2((i0 - L.ly0) | ((i1 - L.ly0) << 16), __float_as_int(w));
  }
  __syncthreads();

  // ---- stage 1: dequantize + scaled IDCT of every ROI block --------------
  const int nbx0 = L.bx1[0] - L.bx0[0] + 1, nby0 = L.by1[0] - L.by0[0] + 1;
  const int nbxc = L.bx1[1] - L.bx0[1] + 1, nbyc = L.by1[1] - L.by0[1] + 1;
  const int nY = nbx0 * nby0, nC = nbxc * nbyc;
  const int total = nY + 2 * nC;
  if constexpr (K == 8) {
    // DC only: v = D(0,0)/8 (all AC basis means vanish exactly), 1 lane/block
    for (int t = tid; t < total; t += kThreads) {
      int c, tt, nbx;
      if (t < nY) { c = 0; tt = t; nbx = nbx0; }
      else { c = 1 + (t - nY) / nC; tt = (t - nY) - (c - 1) * nC; nbx = nbxc; }
      const int by = tt / nbx, bx = tt - by * nbx;
      const int16_t* src = im.coef[c] + (size_t)(L.by0[c] + by) * im.stride[c] + (size_t)(L.bx0[c] + bx) * 64;
      const float d0 = (float)__ldg(src) * qf[c * 64];
      smem[L.off_pl[c] + by * L.pitch[c] + bx] = (uint8_t)round_u8(d0);
    }
  } else {
    const int slot = lane >> 3, r = lane & 7;
    float* sc = scratch + (warp * 4 + slot) * 8 * kScratchPitch;
    for (int base = warp * 4; base < total; base += kWarps * 4) {
      const int t = base + slot;
      const bool act = t < total;
      int c = 0, by = 0, bx = 0;
      float d[8];
      if (act) {
        int tt, nbx;
        if (t < nY) { c = 0; tt = t; nbx = nbx0; }
        else { c = 1 + (t - nY) / nC; tt = (t - nY) - (c - 1) * nC; nbx = nbxc; }
        by = tt / nbx; bx = tt - by * nbx;
        const int16_t* src = im.coef[c] + (size_t)(L.by0[c] + by) * im.stride[c] +
                             (size_t)(L.bx0[c] + bx) * 64 + r * 8;
        const int4 raw = __ldg(reinterpret_cast<const int4*>(src));
        const float4 q0 = *reinterpret_cast<const float4*>(qf + c * 64 + r * 8);
        const float4 q1 = *reinterpret_cast<const float4*>(qf + c * 64 + r * 8 + 4);
        d[0] = (float)(int16_t)(raw.x & 0xffff) * q0.x; d[1] = (float)(raw.x >> 16) * q0.y;
        d[2] = (float)(int16_t)(raw.y & 0xffff) * q0.z; d[3] = (float)(raw.y >> 16) * q0.w;
        d[4] = (float)(int16_t)(raw.z & 0xffff) * q1.x; d[5] = (float)(raw.z >> 16) * q1.y;
        d[6] = (float)(int16_t)(raw.w & 0xffff) * q1.z; d[7] = (float)(raw.w >> 16) * q1.w;
      } else {
#pragma unroll
        for (int i = 0; i < 8; ++i) d[i] = 0.f;
      }
      // row pass: lane r transforms coefficient row v = r along u
      float g[P];
      if constexpr (K == 1) Idct1D<1>::run(d, g);
      else if constexpr (K == 2) Idct1D<2>::run(d, g);
      else Idct1D<4>::run(d, g);
#pragma unroll
      for (int x = 0; x < P; ++x) sc[r * kScratchPitch + x] = g[x];
      __syncwarp();
      // column pass: lane r < P owns output column x = r
      if (act && r < P) {
        float col[8];
#pragma unroll
        for (int v = 0; v < 8; ++v) col[v] = sc[v * kScratchPitch + r];
        float f[P];
        if constexpr (K == 1) Idct1D<1>::run(col, f);
        else if constexpr (K == 2) Idct1D<2>::run(col, f);
        else Idct1D<4>::run(col, f);
        uint8_t* dst = smem + L.off_pl[c] + (by * P) * L.pitch[c] + bx * P + r;
#pragma unroll
        for (int y = 0; y < P; ++y) dst[y * L.pitch[c]] = (uint8_t)round_u8(f[y]);
      }
      __syncwarp();
    }
  }
  __syncthreads();

  if constexpr (DEBUG) {
    for (int c = 0; c < 3; ++c) {
      const int W = c ? im.Wc : im.Wd, H = c ? im.Hc : im.Hd;
      const int y0 = c ? L.cy0 : L.ly0, y1 = c ? L.cy1 : L.ly1;
      const int x0 = c ? L.cx0 : L.lx0, x1 = c ? L.cx1 : L.lx1;
      int16_t* dst = kp.dbg_pl[c] + n * (c ? kp.dbg_stride_c : kp.dbg_stride_y);
      for (int y = y0 + warp; y <= y1; y += kWarps)
        for (int x = x0 + lane; x <= x1; x += 32)
          if (y < H && x < W)
            dst[(size_t)y * W + x] = smem[L.off_pl[c] + (y - L.by0[c] * P) * L.pitch[c] + (x - L.bx0[c] * P)];
    }
  }

  // ---- stage 2: 4:2:0 triangle upsample + YCbCr->RGB over the footprint --
  {
    const uint8_t* Yp = smem + L.off_pl[0];
    const uint8_t* Cbp = smem + L.off_pl[1];
    const uint8_t* Crp = smem + L.off_pl[2];
    const int yorg = L.by0[0] * P, xorg = L.bx0[0] * P;
    const int cyorg = L.by0[1] * P, cxorg = L.bx0[1] * P;
    const int cp = L.pitch[1];
    for (int ry = warp; ry < L.nly; ry += kWarps) {
      const int ly = L.ly0 + ry;
      const int j = ly >> 1;
      const int j2 = min(max((ly & 1) ? j + 1 : j - 1, 0), im.Hc - 1);
      const int rj = (j - cyorg) * cp, rj2 = (j2 - cyorg) * cp;
      const uint8_t* yrow = Yp + (ly - yorg) * L.pitch[0] - xorg;
      uint32_t* orow = rgb + ry * L.nlx - L.lx0;
      for (int lx = L.lx0 + lane; lx <= L.lx1; lx += 32) {
        const int i = lx >> 1;
        const int i2 = min(max((lx & 1) ? i + 1 : i - 1, 0), im.Wc - 1);
        const int ci = i - cxorg, ci2 = i2 - cxorg;
        const int cb = 9 * Cbp[rj + ci] + 3 * (Cbp[rj + ci2] + Cbp[rj2 + ci]) + Cbp[rj2 + ci2];
        const int cr = 9 * Crp[rj + ci] + 3 * (Crp[rj + ci2] + Crp[rj2 + ci]) + Crp[rj2 + ci2];
        const int Y = yrow[lx];
        const int dB = cb - 2048, dR = cr - 2048;
        const uint32_t R = clamp255(Y + jfif_offset(175250 * dR));
        const uint32_t G = clamp255(Y + jfif_offset(-43017 * dB - 89267 * dR));
        const uint32_t B = clamp255(Y + jfif_offset(221500 * dB));
        orow[lx] = R | (G << 8) | (B << 16);
      }
    }
  }
  __syncthreads();

  if constexpr (DEBUG) {
    int16_t* dst = kp.dbg_rgb + n * kp.dbg_stride_rgb;
    for (int ry = warp; ry < L.nly; ry += kWarps)
      for (int rx = lane; rx < L.nlx; rx += 32) {
        const uint32_t v = rgb[ry * L.nlx + rx];
        const size_t o = ((size_t)(L.ly0 + ry) * im.Wd + (L.lx0 + rx)) * 3;
        dst[o] = v & 255; dst[o + 1] = (v >> 8) & 255; dst[o + 2] = (v >> 16) & 255;
      }
  }

  // ---- stage 3: bilinear + normalize + NCHW store -------------------------
  {
    const float na0 = kp.na[0], na1 = kp.na[1], na2 = kp.na[2];
    const float nb0 = kp.nb[0], nb1 = kp.nb[1], nb2 = kp.nb[2];
    const size_t plane = (size_t)kp.OH * OW;
    for (int r = warp; r < oy1 - oy0; r += kWarps) {
      const int2 ty = yt[r];
      const float wy = __int_as_float(ty.y);
      const uint32_t* row0 = rgb + (ty.x & 0xffff) * L.nlx;
      const uint32_t* row1 = rgb + (ty.x >> 16) * L.nlx;
      const size_t obase = ((size_t)n * 3 * kp.OH + (oy0 + r)) * OW;
      for (int ox = lane; ox < OW; ox += 32) {
        const int2 tx = xt[ox];
        const float wx = __int_as_float(tx.y);
        const int x0 = tx.x & 0xffff, x1 = tx.x >> 16;
        const uint32_t p00 = row0[x0], p01 = row0[x1], p10 = row1[x0], p11 = row1[x1];
        float v[3];
#pragma unroll
        for (int ch = 0; ch < 3; ++ch) {
          const float a = (float)((p00 >> (8 * ch)) & 255), b = (float)((p01 >> (8 * ch)) & 255);
          const float cc = (float)((p10 >> (8 * ch)) & 255), dd = (float)((p11 >> (8 * ch)) & 255);
          const float top = fmaf(wx, b - a, a);
          const float bot = fmaf(wx, dd - cc, cc);
          v[ch] = fmaf(wy, bot - top, top);
        }
        const float y0 = fmaf(v[0], na0, nb0), y1 = fmaf(v[1], na1, nb1), y2 = fmaf(v[2], na2, nb2);
        if constexpr (F16) {
          __half* o = reinterpret_cast<__half*>(kp.out) + obase + ox;
          o[0] = __float2half_rn(y0); o[plane] = __float2half_rn(y1); o[2 * plane] = __float2half_rn(y2);
        } else {
          float* o = reinterpret_cast<float*>(kp.out) + obase + ox;
          __stcs(o, y0); __stcs(o + plane, y1); __stcs(o + 2 * plane, y2);
        }
      }
    }
  }
}

}  // namespace smol
