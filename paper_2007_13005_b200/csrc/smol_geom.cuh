// smol_geom.cuh -- per-image and per-tile geometry of the fused Smol
// preprocessing kernel, shared by the host runtime (validation, shared-memory
// sizing, smol_debug_geometry) and the device kernels.  Part of the CUDA path
// only; the oracle (oracle/) has its own, independent implementation.
#pragma once
#include <stdint.h>

#if defined(__CUDACC__)
#define SMOL_HD __host__ __device__ __forceinline__
#else
#define SMOL_HD inline
#endif

namespace smol {

// Threads per CTA: the kernel is instantiated for 256 (3 CTAs per SM), 192
// (4 CTAs per SM, used when the tile's shared memory allows 4) and 128 (6
// CTAs per SM, small footprints: thumbnails, reduced-scale decodes, where a
// CTA's serial prologue/barrier latency dominates and more CTAs per SM hide
// it); all keep 24 warps per SM at <= 80 registers per thread.
constexpr int kThreadsWide = 256, kThreadsNarrow = 192, kThreadsTiny = 128;
constexpr int kStepRows = 16;             // decoded luma rows per rolling step (one MCU row at scale 1)
constexpr int kYRing = 32;                // luma rows kept in smem (two steps)
constexpr int kCRing = 16;                // chroma rows kept per component (two steps)
// RGB rows kept: output(s) reads rows [ready_{s-1}, ready_s + 1] after
// colour(s) wrote (ready_{s-1}, ready_s] (+ one garbage row at the footprint
// ends); ready_s - ready_{s-1} <= 18, so 20 rows never alias a live row.
constexpr int kRgbRing = 20;

SMOL_HD int ceil_div(int a, int b) { return (a + b - 1) / b; }
SMOL_HD int imin(int a, int b) { return a < b ? a : b; }
SMOL_HD int imax(int a, int b) { return a > b ? a : b; }

// Device-side image descriptor (built by the host in smol_preproc_run).
struct __align__(16) DevImage {
  const int16_t* coef[3];   // block-raster [bh][bw][64] int16, natural order
  int32_t stride[3];        // int16 elements per block row
  int32_t qidx[3];          // quant table index per component
  int32_t nbw[3];           // valid block columns per component: ceil(W/8), ceil(W/16)
  int32_t Wd, Hd;           // decoded luma size at scale 1/k (R4)
  int32_t Wc, Hc;           // decoded chroma size
  int32_t Wr, Hr;           // resized size
  int32_t left, top;        // crop origin in resized coordinates
  int32_t gray;             // 1: one component (subsampling 400): no chroma blocks, Cb = Cr = 128
  int32_t sx0, sy0, sw, sh; // source window of the resize in decoded luma px: the whole
                            // image (0, 0, Wd, Hd), or an ROI rectangle's window (R15)
  int32_t hs, vs;           // chroma factors of the decoded planes (T.81 A.1.1): 2,2 =
                            // 4:2:0 (and gray); 2,1 = 4:2:2; 1,1 = 4:4:4, and 4:2:0
                            // decoded with chroma at twice the scale (R18)
  int32_t ck;               // decode scale denominator of the chroma blocks (K, or K/2)
  int32_t pad_;
};

// Per-image reference of a run (32 B): the image's coefficient planes and
// the index of its "kind" -- the DevImage holding everything else, shared by
// consecutive images with equal descriptors (a batch of equal-size images
// has one kind, so the host writes and uploads 32 B per image).
struct __align__(16) DevRef {
  const int16_t* coef[3];
  int32_t kind;
  int32_t pad_;
};

// Reading R9: the half-pixel bilinear source index of destination index d
// (R8: src = max(0, (d + 1/2) in/out - 1/2)), from exact integers:
//   num = max(0, (2d+1) in - out),  i0 = num div 2out,  w = (num mod 2out) / 2out,
//   i1 = min(i0 + 1, in - 1).
SMOL_HD void src_tap(int d, int in, int out, int& i0, int& i1, float& w) {
  long long num = (long long)(2 * d + 1) * in - out;
  if (num < 0) num = 0;
  const long long den = 2LL * out;
  if (num < (1LL << 32)) {
    // 32-bit unsigned division (the common case; the 64-bit one is a long
    // software routine on the GPU)
    const uint32_t n32 = (uint32_t)num, d32 = (uint32_t)den, q32 = n32 / d32;
    i0 = (int)q32;
    w = (float)(n32 - q32 * d32) / (float)d32;   // both exact in fp32 (< 2^24)
  } else {
    const long long q = num / den;
    i0 = (int)q;
    w = (float)(num - q * den) / (float)den;
  }
  if (i0 > in - 1) i0 = in - 1;
  i1 = imin(i0 + 1, in - 1);
}

// Taps of the resize of an image's source window (the whole decoded image,
// or an ROI rectangle's window): R9 within the window, then offset to
// decoded coordinates.
SMOL_HD void src_tap_x(const DevImage& im, int d, int& i0, int& i1, float& w) {
  src_tap(d, im.sw, im.Wr, i0, i1, w);
  i0 += im.sx0; i1 += im.sx0;
}
SMOL_HD void src_tap_y(const DevImage& im, int d, int& i0, int& i1, float& w) {
  src_tap(d, im.sh, im.Hr, i0, i1, w);
  i0 += im.sy0; i1 += im.sy0;
}

SMOL_HD int align16(int x) { return (x + 15) & ~15; }

// RGB ring slot of decoded row r >= 0 (kRgbRing is even, so an even row's
// odd neighbour never wraps)
SMOL_HD int rgb_slot(int r) { return (int)((uint32_t)r % (uint32_t)kRgbRing); }

// Shared-memory rings (fixed pitches so neighbour loads use immediate offsets):
//   Y   : kYRing slots x kYP bytes, column = x - xbase[0]
//   Cb/Cr: kCSlots = 16 + 2 slots x kCP bytes each; row r lives in slot
//          (r & 15) + 1, slot 0 mirrors slot 16 and slot 17 mirrors slot 1, so
//          rows j-1, j, j+1 are always at constant stride; column
//          c - xbase[c] + kCPad (image-edge columns replicated into the pad)
//   RGB : kRgbRing + 1 slots (row r in slot r mod kRgbRing; the last slot mirrors slot 0) x rgb_p u32
// Ring pitches come in two compile-time configurations (kernel template
// parameter YP, chroma pitch YP/2): wide (512), narrow (384, fits 4 CTAs
// per SM for footprints up to ~370 decoded columns) and tiny (128, footprints
// up to ~110 decoded columns).
constexpr int kYPWide = 512, kYPNarrow = 384, kYPTiny = 128;
// RGB ring pitch (u32): yp - kRgbPitchPad, which is 4 (mod 32) so that rows
// r and r+1 start in different shared-memory banks
#ifndef SMOL_RGB_PITCH_PAD
#define SMOL_RGB_PITCH_PAD 28
#endif
__host__ __device__ constexpr int rgb_pitch(int yp) { return yp - SMOL_RGB_PITCH_PAD; }
constexpr int kCPad = 8;
constexpr int kCSlots = 18;
// Generic-chroma kernels (4:2:2 / 4:4:4 / mixed batches; template flag GC):
// chroma rings as tall and as wide as the luma ring (vertically
// unsubsampled chroma advances 16 rows per step, horizontally unsubsampled
// chroma is as wide as luma): 32 rows + 2 guard slots, pitch yp.
constexpr int kCRingG = 32;
constexpr int kCSlotsG = kCRingG + 2;
__host__ __device__ constexpr int c_ring(bool gc) { return gc ? kCRingG : kCRing; }
__host__ __device__ constexpr int c_slots(bool gc) { return gc ? kCSlotsG : kCSlots; }
__host__ __device__ constexpr int c_pitch(int yp, bool gc) { return gc ? yp : yp / 2; }
__host__ __device__ constexpr int off_c(int yp) { return kYRing * yp; }                  // Cb ring, then Cr ring (Y ring at 0)
__host__ __device__ constexpr int off_q(int yp, bool gc = false) {                         // dequant tables (3 x 64 float)
  return off_c(yp) + 2 * c_slots(gc) * c_pitch(yp, gc);
}
__host__ __device__ constexpr int off_rgb(int yp, bool gc = false) { return off_q(yp, gc) + 3 * 64 * 4; }  // RGB ring (size depends on the tile)

// Magic-number division: exact for n * d < 2^32 (the host caps the tile
// height so every kernel division meets it).
struct FastDiv {
  uint32_t d, m;
};
SMOL_HD FastDiv make_fastdiv(uint32_t d) { return FastDiv{d, d <= 1 ? 0u : (uint32_t)(0xFFFFFFFFu / d) + 1u}; }

struct TileLayout {
  int oy0, oy1, ox0, ox1;          // output tile
  int ly0, ly1, lx0, lx1;          // luma (decoded) tap footprint, inclusive
  int cy0, cy1, cx0, cx1;          // chroma footprint incl. triangle neighbours (R2)
  int by0[3], by1[3], bx0[3], bx1[3];   // ROI block ranges per component
  int xbase[3];                    // decoded column of ring column 0 (= bx0 * P)
  int rgb_x0, rgb_w, rgb_p;        // RGB ring: first column, width, pitch (u32; rgb_pitch(yp), compile-time in the kernel)
  int r0, nsteps;                  // first rolling-step row (16-aligned) and step count
  int fits;                        // footprint fits the fixed ring pitches
  int tap_off;                     // int4 index of the host-computed tap region (-1: computed by the CTA)
  // byte offsets in dynamic shared memory
  int off_q, off_xt, off_yt, off_st, off_y, off_c, off_rgb, total;
  // the kernel's task-index divisors: luma / chroma blocks per block row,
  // 4-column colour tasks per quad row, 4-pixel output quads per row
  FastDiv fd_y, fd_c, fd_t4, fd_q4;
  FastDiv fd_fw, fd_cw;            // luma / chroma footprint widths (thumbnail kernel)
};

SMOL_HD void tile_layout(const DevImage& im, int K, int oy0, int oy1, int ox0, int ox1, TileLayout& L,
                         int yp = kYPWide, bool gc = false) {
  const int P = 8 / K;
  int a, b; float w;
  L.oy0 = oy0; L.oy1 = oy1; L.ox0 = ox0; L.ox1 = ox1;
  src_tap_x(im, im.left + ox0, L.lx0, b, w);
  src_tap_x(im, im.left + ox1 - 1, a, L.lx1, w);
  src_tap_y(im, im.top + oy0, L.ly0, b, w);
  src_tap_y(im, im.top + oy1 - 1, a, L.ly1, w);
  // chroma rows/cols used by the centred triangle filter of luma rows
  // [ly0, ly1] along a subsampled axis: floor((ly0-1)/2) .. floor((ly1+1)/2),
  // clamped (reading R2); along an unsubsampled axis the same rows
  L.cy0 = im.vs == 2 ? imax(0, (L.ly0 - 1) >> 1) : imin(L.ly0, im.Hc - 1);
  L.cy1 = imin(im.Hc - 1, im.vs == 2 ? (L.ly1 + 1) >> 1 : L.ly1);
  L.cx0 = im.hs == 2 ? imax(0, (L.lx0 - 1) >> 1) : imin(L.lx0 & ~3, im.Wc - 1);
  L.cx1 = imin(im.Wc - 1, im.hs == 2 ? (L.lx1 + 1) >> 1 : (L.lx1 | 3));
  // luma columns are processed 4 at a time (two 2x2 quads): widen to
  // 4-alignment (never beyond the image's valid block columns)
  L.by0[0] = L.ly0 / P; L.by1[0] = L.ly1 / P;
  L.bx0[0] = (L.lx0 & ~3) / P;
  L.bx1[0] = imin((L.lx1 | 3) / P, im.nbw[0] - 1);
  const int PC = 8 / (im.ck > 0 ? im.ck : K);   // chroma samples per block side
  for (int c = 1; c < 3; ++c) {
    L.by0[c] = L.cy0 / PC; L.by1[c] = L.cy1 / PC;
    L.bx0[c] = L.cx0 / PC; L.bx1[c] = L.cx1 / PC;
  }
  // grayscale: no chroma block rows (the kernel fills the chroma rings with
  // 128, the neutral value, so colour conversion gives R = G = B = Y)
  if (im.gray)
    for (int c = 1; c < 3; ++c) L.by1[c] = L.by0[c] - 1;
  for (int c = 0; c < 3; ++c) L.xbase[c] = L.bx0[c] * (c ? PC : P);
  L.rgb_x0 = L.lx0 & ~3;
  L.rgb_w = ((L.lx1 | 3) - L.rgb_x0 + 1);
  L.rgb_p = rgb_pitch(yp);         // fixed pitch (u32): row r+1 is an immediate offset from row r
  L.r0 = L.ly0 & ~(kStepRows - 1);
  // the last step must cover luma row ly1 and chroma row cy1 (luma vs cy1)
  L.nsteps = ((imax(L.ly1, im.vs * L.cy1) - L.r0) / kStepRows) + 1;
  L.fits = ((L.bx1[0] - L.bx0[0] + 1) * P + 4 <= yp) &&
           ((L.bx1[1] - L.bx0[1] + 1) * PC + 2 * kCPad <= c_pitch(yp, gc)) && (L.rgb_w + 4 <= L.rgb_p) &&
           (gc || (im.hs == 2 && im.vs == 2));
  int off = 0;
  // fixed-size regions first, at compile-time offsets (kOff*), so the hot
  // loops address them as immediates instead of keeping base pointers live
  L.off_y = 0;
  L.off_c = off_c(yp);
  L.off_q = off_q(yp, gc);
  L.off_rgb = off_rgb(yp, gc);
  off = off_rgb(yp, gc) + align16(L.rgb_p * 4 * (kRgbRing + 1));
  L.off_xt = off;  off += ((ox1 - ox0 + 3) >> 2) * 32;       // x taps per pixel pair: {4 x0 a, 4 x0 b, w a, w b}
  L.off_yt = off;  off += align16((oy1 - oy0) * 8);           // y taps: {ring byte offset of row y0 | y1<<16, w}
  L.off_st = off;  off += align16(L.nsteps * 8);              // per-step {ready, done}
  L.total = off;
  L.tap_off = -1;
  L.fd_y = make_fastdiv(L.bx1[0] - L.bx0[0] + 1);
  L.fd_c = make_fastdiv(L.bx1[1] - L.bx0[1] + 1);
  L.fd_t4 = make_fastdiv(L.rgb_w >> 2);
  L.fd_q4 = make_fastdiv((ox1 - ox0 + 3) >> 2);
  L.fd_fw = make_fastdiv(L.lx1 - L.lx0 + 1);
  L.fd_cw = make_fastdiv(L.cx1 - L.cx0 + 1);
}

// Bilinear taps of a tile, in the layout of its shared-memory tap region
// [off_xt, off_st) (computed per CTA, or once per (image kind, tile) by the
// host and copied in -- the same function either way, so the same bits).
// x entry i (output column ox0 + i, padded to a multiple of 4): pixel pairs
// {byte offset of x0 (a), (b), w (a), w (b)}; output quad q reads pair A at
// int4 [q] and pair B at [nq4 + q]; a clamped upper tap gets weight 0.
SMOL_HD void tile_xtap(const DevImage& im, const TileLayout& L, int i, int* xt) {
  const int ntw = L.ox1 - L.ox0, nq4 = (ntw + 3) >> 2;
  int i0, i1; float w;
  src_tap_x(im, im.left + L.ox0 + (i < ntw - 1 ? i : ntw - 1), i0, i1, w);
  int* e = xt + (((i >> 1) & 1) * nq4 + (i >> 2)) * 4 + (i & 1);
  e[0] = (i0 - L.rgb_x0) * 4;
  union { float f; int i; } u;
  u.f = i1 == i0 ? 0.f : w;
  e[2] = u.i;
}
// y entry i (output row oy0 + i): {byte offset of RGB ring row i0 | i1 << 16, w}
SMOL_HD void tile_ytap(const DevImage& im, const TileLayout& L, int i, int pitch4, int* yt) {
  int i0, i1; float w;
  src_tap_y(im, im.top + L.oy0 + i, i0, i1, w);
  union { float f; int i; } u;
  u.f = i1 == i0 ? 0.f : w;
  yt[2 * i] = (rgb_slot(i0) * pitch4) | (i1 << 16);
  yt[2 * i + 1] = u.i;
}
// bytes of the tap region (x taps then y taps)
SMOL_HD int tile_tap_bytes(const TileLayout& L) { return L.off_st - L.off_xt; }

// Thumbnail kernel taps (one tile = the whole output): column pair q {4 x0
// (a), 4 x0 (b), w (a), w (b)} relative to the footprint, and row i
// {y0 - ly0 | (y1 - ly0) << 16, w}.
SMOL_HD void thumb_xp(const DevImage& im, const TileLayout& L, int OW, int q, int* e) {
  int a0, a1, b0, b1; float wa, wb;
  src_tap_x(im, im.left + 2 * q, a0, a1, wa);
  src_tap_x(im, im.left + (2 * q + 1 < OW - 1 ? 2 * q + 1 : OW - 1), b0, b1, wb);
  union { float f; int i; } u, v;
  u.f = a1 == a0 ? 0.f : wa;
  v.f = b1 == b0 ? 0.f : wb;
  e[0] = 4 * (a0 - L.lx0); e[1] = 4 * (b0 - L.lx0); e[2] = u.i; e[3] = v.i;
}
SMOL_HD void thumb_yt(const DevImage& im, const TileLayout& L, int i, int* e) {
  int i0, i1; float w;
  src_tap_y(im, im.top + i, i0, i1, w);
  union { float f; int i; } u;
  u.f = i1 == i0 ? 0.f : w;
  e[0] = (i0 - L.ly0) | ((i1 - L.ly0) << 16);
  e[1] = u.i;
}
// int4 words of a thumbnail tap region: (OW+1)/2 column pairs, then OH rows (2 per int4)
SMOL_HD int thumb_tap_words(int OW, int OH) { return ((OW + 1) >> 1) + ((OH + 1) >> 1); }

SMOL_HD long long tile_roi_blocks(const TileLayout& L) {
  long long n = 0;
  for (int c = 0; c < 3; ++c) n += (long long)(L.by1[c] - L.by0[c] + 1) * (L.bx1[c] - L.bx0[c] + 1);
  return n;
}

// Last RGB row produced after rolling step s (decoded luma rows
// [r0 + 16 s, r0 + 16 s + 16) and chroma rows [.. /2, +8) are decoded):
// luma row L needs chroma rows L>>1 and, for odd L, min(L>>1 + 1, Hc - 1).
// While chroma is the limit the step ends on an odd row (2 chi - 1), so the
// next step starts on an even row and 2x2 quads never straddle steps.
SMOL_HD int ready_after(const TileLayout& L, int Hc, int s, int vs = 2) {
  const int R = L.r0 + kStepRows * s;
  int r = imin(L.ly1, R + kStepRows - 1);
  if (vs == 1) return r;             // unsubsampled rows: luma row L needs chroma row L only
  const int chi = imin(L.cy1, (R >> 1) + kStepRows / 2 - 1);
  if (chi < Hc - 1) r = imin(r, chi < L.cy1 ? 2 * chi - 1 : 2 * chi);
  return r;
}


}  // namespace smol
