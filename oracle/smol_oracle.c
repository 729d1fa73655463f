/*
 * smol_oracle.c -- plain, slow CPU oracle (TEST INFRASTRUCTURE ONLY; see
 * smol_oracle.h).  Written from the paper and the readings in DESIGN.md; no
 * blocking, fusion, ROI or reordering.  Direct 2-D IDCT sum (4096 MACs per
 * 8x8 block at scale 1), whole-image decode, whole-image resize, then crop.
 *
 * Parity pins: tests/test_oracle_*.py (scipy idctn, torch bilinear, Fraction
 * colour arithmetic, libjpeg-turbo jidctred constants, SURVEY worked pins).
 */
#include "smol_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

static const double ORACLE_PI = 3.14159265358979323846;

/* ------------------------------------------------------------------ IDCT --
 * T.81 A.3.3 (inverse DCT):
 *   s(y,x) = 1/4 sum_u sum_v C(u) C(v) S(v,u) cos((2x+1)u pi/16) cos((2y+1)v pi/16)
 * with C(0) = 1/sqrt2, C(u>0) = 1.  Writing t(u,x) = sqrt2 C(u) cos((2x+1)u pi/16)
 * this is  s(y,x) = 1/8 sum_v sum_u S(v,u) t(v,y) t(u,x).  t is exactly 1 for
 * u = 0 and exactly +-1 for u = 4 (sqrt2 cos((2x+1)pi/4) = +-1); those entries
 * are stored exactly so that exact half-integer ties (DC-only and {0,4}
 * blocks) stay exact (reading R3). */
static double oracle_t(int u, int x) {
  if (u == 0) return 1.0;
  if (u == 4) {
    int m = (2 * x + 1) % 8;          /* angle (2x+1) pi/4 */
    return (m == 1 || m == 7) ? 1.0 : -1.0;
  }
  return sqrt(2.0) * cos((double)((2 * x + 1) * u) * ORACLE_PI / 16.0);
}

/* Reading R1 (Definition A): at scale 1/k each output sample is the mean of
 * the k x k box of the unrounded 8x8 IDCT.  By linearity the box mean of
 * 1/8 sum D t(v,y) t(u,x) is 1/8 sum D a_k(v,i) a_k(u,j) with the box-averaged
 * basis  a_k(u,j) = 1/k sum_{x=jk}^{jk+k-1} t(u,x)  (a_1 = t).
 * By the sum-of-cosines identity
 *   sum_{m<k} cos(theta0 + m u pi/8) = sin(k u pi/16)/sin(u pi/16) cos(k u (2j+1) pi/16)
 * a_k(u,j) is exactly zero for u > 0 when k*u = 0 (mod 16) or
 * k*u*(2j+1) = 8 (mod 16) (e.g. u = 4 at k = 2; u in {2,4,6} at k = 4; every
 * u > 0 at k = 8).  Such entries are stored as exact zeros, like the exact
 * +-1 entries of t, so that DC/8 ties stay exact at every scale. */
static double oracle_a(int k, int u, int j) {
  if (u > 0 && ((k * u) % 16 == 0 || (k * u * (2 * j + 1)) % 16 == 8)) return 0.0;
  double s = 0.0;
  for (int x = j * k; x < j * k + k; ++x) s += oracle_t(u, x);
  return s / (double)k;
}

/* Reading R16 (Definition B, the alternative of R1): at scale 1/k, with
 * N = 8/k, the N x N output is the orthonormal N-point 2-D IDCT of the
 * top-left N x N coefficients scaled by N/8 (the N-point DCT of a block's
 * low-pass content is sqrt(N/8) times the 8-point one per axis; libjpeg >= 7
 * jpeg_idct_NxN).  Orthonormal N-point IDCT:
 *   f(i,j) = sum_v sum_u alpha(v) alpha(u) F(v,u) cos((2i+1)v pi/2N) cos((2j+1)u pi/2N),
 *   alpha(0) = sqrt(1/N), alpha(u>0) = sqrt(2/N);  with F = (N/8) D this is
 *   f(i,j) = 1/8 sum_v sum_u D(v,u) b_N(v,i) b_N(u,j),
 *   b_N(u,x) = sqrt2 C(u) cos((2x+1) u pi / 2N)   (b_8 = t).
 * b_N(0,x) = 1 and b_N(N/2,x) = sqrt2 cos((2x+1) pi/4) = +-1 exactly; those
 * entries are stored exactly (DC and u = N/2 ties stay exact, R3).  At N = 1
 * (k = 8) this is DC/8, Definition A's value. */
static double oracle_b(int N, int u, int x) {
  if (u == 0) return 1.0;
  if (2 * u == N) {
    int m = (2 * x + 1) % 8;          /* angle (2x+1) pi/4 */
    return (m == 1 || m == 7) ? 1.0 : -1.0;
  }
  return sqrt(2.0) * cos((double)((2 * x + 1) * u) * ORACLE_PI / (2.0 * N));
}

/* Dequantize (D = coef * Q, "inverse transform") and decode one
 * block at scale 1/k: v[i*P+j] = 1/8 sum_v sum_u D(v,u) a_k(v,i) a_k(u,j),
 * P = 8/k samples per side, before the level shift (Definition A); with
 * def = 1 the basis is b_P over u, v < P (Definition B, zero elsewhere). */
static void oracle_idct_block_def(const int16_t* coef, const uint16_t* q, int k, int def, double* v) {
  const int P = 8 / k;
  double a[8][8];
  long long D[64];
  for (int u = 0; u < 8; ++u)
    for (int j = 0; j < P; ++j)
      a[u][j] = def == 0 ? oracle_a(k, u, j) : (u < P ? oracle_b(P, u, j) : 0.0);
  for (int i = 0; i < 64; ++i) D[i] = (long long)coef[i] * (long long)q[i];
  for (int i = 0; i < P; ++i)
    for (int j = 0; j < P; ++j) {
      double s = 0.0;
      for (int vv = 0; vv < 8; ++vv)
        for (int u = 0; u < 8; ++u) s += (double)D[vv * 8 + u] * a[vv][i] * a[u][j];
      v[i * P + j] = s / 8.0;
    }
}


/* Reading R3: u8 = clamp(floor(v + 128 + 1/2), 0, 255) (round half up). */
static uint8_t oracle_round_u8(double v) {
  double r = floor(v + 128.0 + 0.5);
  if (r < 0.0) return 0;
  if (r > 255.0) return 255;
  return (uint8_t)r;
}

int oracle_decode_plane(const oracle_plane* pl, int32_t k, int32_t out_w, int32_t out_h,
                        double* v_out, uint8_t* u8_out) {
  return oracle_decode_plane2(pl, k, 0, out_w, out_h, v_out, u8_out);
}

int oracle_decode_plane2(const oracle_plane* pl, int32_t k, int32_t idct_def, int32_t out_w,
                         int32_t out_h, double* v_out, uint8_t* u8_out) {
  if (!pl || !pl->coef || !pl->q || !u8_out) return 1;
  if (idct_def != 0 && idct_def != 1) return 4;
  if (k != 1 && k != 2 && k != 4 && k != 8) return 2;
  const int P = 8 / k;                      /* output samples per block side */
  const int nbx = (out_w + P - 1) / P, nby = (out_h + P - 1) / P;
  if (nbx > pl->blocks_w || nby > pl->blocks_h) return 3;
  double v[64];
  for (int by = 0; by < nby; ++by)
    for (int bx = 0; bx < nbx; ++bx) {
      const int16_t* blk = pl->coef + (size_t)by * pl->row_stride + (size_t)bx * 64;
      oracle_idct_block_def(blk, pl->q, k, idct_def, v);
      for (int i = 0; i < P; ++i)
        for (int j = 0; j < P; ++j) {
          int y = by * P + i, x = bx * P + j;
          if (y >= out_h || x >= out_w) continue;
          if (v_out) v_out[(size_t)y * out_w + x] = v[i * P + j];
          u8_out[(size_t)y * out_w + x] = oracle_round_u8(v[i * P + j]);
        }
    }
  return 0;
}

/* ------------------------------------------------------------ colour ------
 * JFIF 1.02 (reading R6), chroma given in 1/16 units c16 (Cb = c16/16):
 *   R = Y + 1.402 (Cr - 128)
 *   G = Y - 0.344136 (Cb - 128) - 0.714136 (Cr - 128)
 *   B = Y + 1.772 (Cb - 128)
 * evaluated exactly over the common denominator 16*10^6, then rounded half
 * up and clamped to [0, 255]. */
static long long oracle_floor_div(long long a, long long b) {   /* b > 0 */
  long long q = a / b;
  if ((a % b) != 0 && a < 0) q -= 1;
  return q;
}
static uint8_t oracle_clamp_u8(long long x) {
  return (uint8_t)(x < 0 ? 0 : (x > 255 ? 255 : x));
}
void oracle_color(int32_t Y, int32_t cb16, int32_t cr16, uint8_t rgb[3]) {
  const long long den = 16000000LL;               /* 16 * 10^6 */
  long long dcb = (long long)cb16 - 2048;         /* 16 (Cb - 128) */
  long long dcr = (long long)cr16 - 2048;
  long long y = (long long)Y * den;
  long long r = y + 1402000LL * dcr;              /* 1.402   * 10^6 */
  long long g = y - 344136LL * dcb - 714136LL * dcr;
  long long b = y + 1772000LL * dcb;              /* 1.772   * 10^6 */
  rgb[0] = oracle_clamp_u8(oracle_floor_div(r + den / 2, den));
  rgb[1] = oracle_clamp_u8(oracle_floor_div(g + den / 2, den));
  rgb[2] = oracle_clamp_u8(oracle_floor_div(b + den / 2, den));
}

/* Reading R2: 2x centred ("triangle") upsampling of 4:2:0 chroma.  Luma
 * sample (2j+b, 2i+a) takes 9/16 C[j][i] + 3/16 C[j][i'] + 3/16 C[j'][i]
 * + 1/16 C[j'][i'] with i' = i-1 (a=0) or i+1 (a=1), j' likewise; indices
 * clamped to the valid chroma size.  Kept exact in 1/16 units. */
static int32_t oracle_upsample_at(const uint8_t* C, int32_t Wc, int32_t Hc, int32_t X, int32_t Yr) {
  int32_t i = X / 2, j = Yr / 2;
  int32_t i2 = (X % 2 == 0) ? i - 1 : i + 1;
  int32_t j2 = (Yr % 2 == 0) ? j - 1 : j + 1;
  if (i2 < 0) i2 = 0;
  if (i2 > Wc - 1) i2 = Wc - 1;
  if (j2 < 0) j2 = 0;
  if (j2 > Hc - 1) j2 = Hc - 1;
  if (i > Wc - 1) i = Wc - 1;
  if (j > Hc - 1) j = Hc - 1;
  return 9 * C[(size_t)j * Wc + i] + 3 * C[(size_t)j * Wc + i2] +
         3 * C[(size_t)j2 * Wc + i] + 1 * C[(size_t)j2 * Wc + i2];
}

/* Reading R2 per axis (4:2:2, 4:4:4 and 4:2:0): along an axis subsampled by
 * 2, luma position X takes 3/4 C[X/2] + 1/4 C[X/2 -+ 1] (- for even X, +
 * for odd), clamped to the valid chroma size; along an axis that is not
 * subsampled it takes C[X] (weight 4/4).  The 2-D value is the product of
 * the two axis filters, kept exact in 1/16 units (4:2:0: 9/3/3/1, as above). */
static void oracle_axis_taps(int32_t X, int32_t f, int32_t n, int32_t* i, int32_t* i2, int32_t* w, int32_t* w2) {
  if (f == 1) {
    *i = X < n ? X : n - 1; *i2 = *i; *w = 4; *w2 = 0;
    return;
  }
  *i = X / 2;
  *i2 = (X % 2 == 0) ? *i - 1 : *i + 1;
  if (*i2 < 0) *i2 = 0;
  if (*i2 > n - 1) *i2 = n - 1;
  if (*i > n - 1) *i = n - 1;
  *w = 3; *w2 = 1;
}
static int32_t oracle_upsample_at2(const uint8_t* C, int32_t Wc, int32_t Hc, int32_t X, int32_t Yr,
                                   int32_t hs, int32_t vs) {
  int32_t i, i2, wx, wx2, j, j2, wy, wy2;
  oracle_axis_taps(X, hs, Wc, &i, &i2, &wx, &wx2);
  oracle_axis_taps(Yr, vs, Hc, &j, &j2, &wy, &wy2);
  return wy * (wx * C[(size_t)j * Wc + i] + wx2 * C[(size_t)j * Wc + i2]) +
         wy2 * (wx * C[(size_t)j2 * Wc + i] + wx2 * C[(size_t)j2 * Wc + i2]);
}

int oracle_upsample_color(const uint8_t* Y, int32_t Wd, int32_t Hd,
                          const uint8_t* Cb, const uint8_t* Cr, int32_t Wc, int32_t Hc,
                          int32_t* c16_out, uint8_t* rgb_out) {
  if (!Y || !Cb || !Cr || !rgb_out || Wd <= 0 || Hd <= 0 || Wc <= 0 || Hc <= 0) return 1;
  for (int32_t y = 0; y < Hd; ++y)
    for (int32_t x = 0; x < Wd; ++x) {
      int32_t cb = oracle_upsample_at(Cb, Wc, Hc, x, y);
      int32_t cr = oracle_upsample_at(Cr, Wc, Hc, x, y);
      if (c16_out) {
        c16_out[((size_t)y * Wd + x) * 2 + 0] = cb;
        c16_out[((size_t)y * Wd + x) * 2 + 1] = cr;
      }
      oracle_color(Y[(size_t)y * Wd + x], cb, cr, rgb_out + ((size_t)y * Wd + x) * 3);
    }
  return 0;
}

int oracle_upsample_color2(const uint8_t* Y, int32_t Wd, int32_t Hd,
                           const uint8_t* Cb, const uint8_t* Cr, int32_t Wc, int32_t Hc,
                           int32_t hs, int32_t vs, int32_t* c16_out, uint8_t* rgb_out) {
  if (!Y || !Cb || !Cr || !rgb_out || Wd <= 0 || Hd <= 0 || Wc <= 0 || Hc <= 0) return 1;
  if ((hs != 1 && hs != 2) || (vs != 1 && vs != 2)) return 2;
  for (int32_t y = 0; y < Hd; ++y)
    for (int32_t x = 0; x < Wd; ++x) {
      int32_t cb = oracle_upsample_at2(Cb, Wc, Hc, x, y, hs, vs);
      int32_t cr = oracle_upsample_at2(Cr, Wc, Hc, x, y, hs, vs);
      if (c16_out) {
        c16_out[((size_t)y * Wd + x) * 2 + 0] = cb;
        c16_out[((size_t)y * Wd + x) * 2 + 1] = cr;
      }
      oracle_color(Y[(size_t)y * Wd + x], cb, cr, rgb_out + ((size_t)y * Wd + x) * 3);
    }
  return 0;
}

/* ------------------------------------------------------------- fp16 ------ */
uint16_t oracle_f64_to_f16(double x) {
  uint16_t sign = (uint16_t)(signbit(x) ? 0x8000u : 0u);
  double a = fabs(x);
  if (isnan(x)) return 0x7e00u;
  if (a >= 65520.0) return (uint16_t)(sign | 0x7c00u);       /* overflow -> inf */
  if (a < ldexp(1.0, -14)) {                                  /* subnormal range */
    double m = a / ldexp(1.0, -24);                           /* units of 2^-24 */
    double r = nearbyint(m);                                  /* RNE (default mode) */
    return (uint16_t)(sign | (uint16_t)r);
  }
  int e;
  double f = frexp(a, &e);          /* a = f * 2^e, f in [0.5, 1) */
  double m = ldexp(f, 11);          /* [1024, 2048) */
  double r = nearbyint(m);
  if (r >= 2048.0) { r = 1024.0; e += 1; }
  int be = e - 1 + 15;              /* biased exponent: a = (r/1024) * 2^(e-1) */
  if (be >= 31) return (uint16_t)(sign | 0x7c00u);
  return (uint16_t)(sign | (uint16_t)(be << 10) | (uint16_t)((int)r - 1024));
}

/* --------------------------------------------------------------- resize ---
 * Reading R8: half-pixel bilinear, align_corners = False, no antialias:
 *   src = max(0, (d + 1/2) * in / out - 1/2),  i0 = floor(src),
 *   i1 = min(i0 + 1, in - 1),  w = src - i0.
 * The whole image is resized ("resize the image ... short edge 256"),
 * then the crop window is taken ("centrally crop"). */
static void oracle_src_index(int32_t d, int32_t in, int32_t out, int32_t* i0, int32_t* i1, double* w) {
  double src = ((double)d + 0.5) * (double)in / (double)out - 0.5;
  if (src < 0.0) src = 0.0;
  double f = floor(src);
  *i0 = (int32_t)f;
  if (*i0 > in - 1) *i0 = in - 1;
  *i1 = (*i0 + 1 < in) ? *i0 + 1 : in - 1;
  *w = src - (double)*i0;
}

int oracle_resize_crop_normalize(const uint8_t* rgb, int32_t Wd, int32_t Hd,
                                 int32_t Wr, int32_t Hr, int32_t left, int32_t top,
                                 int32_t OW, int32_t OH, const double mean[3],
                                 const double std[3], int32_t out_f16, void* out,
                                 double* resized_out) {
  if (!rgb || !out || Wd <= 0 || Hd <= 0 || Wr <= 0 || Hr <= 0) return 1;
  if (left < 0 || top < 0 || left + OW > Wr || top + OH > Hr) return 2;
  double* full = (double*)malloc(sizeof(double) * (size_t)Wr * Hr * 3);
  if (!full) return 3;
  for (int32_t ry = 0; ry < Hr; ++ry) {
    int32_t y0, y1; double wy;
    oracle_src_index(ry, Hd, Hr, &y0, &y1, &wy);
    for (int32_t rx = 0; rx < Wr; ++rx) {
      int32_t x0, x1; double wx;
      oracle_src_index(rx, Wd, Wr, &x0, &x1, &wx);
      for (int c = 0; c < 3; ++c) {
        double p00 = rgb[((size_t)y0 * Wd + x0) * 3 + c], p01 = rgb[((size_t)y0 * Wd + x1) * 3 + c];
        double p10 = rgb[((size_t)y1 * Wd + x0) * 3 + c], p11 = rgb[((size_t)y1 * Wd + x1) * 3 + c];
        double top_ = (1.0 - wx) * p00 + wx * p01;
        double bot_ = (1.0 - wx) * p10 + wx * p11;
        full[((size_t)c * Hr + ry) * Wr + rx] = (1.0 - wy) * top_ + wy * bot_;
      }
    }
  }
  /* crop, then P:376-378: convert to float, /255, subtract mean, divide by
   * std; channels-first. */
  for (int c = 0; c < 3; ++c)
    for (int32_t oy = 0; oy < OH; ++oy)
      for (int32_t ox = 0; ox < OW; ++ox) {
        double x = full[((size_t)c * Hr + (oy + top)) * Wr + (ox + left)];
        size_t o = ((size_t)c * OH + oy) * OW + ox;
        if (resized_out) resized_out[o] = x;
        double yv = (x / 255.0 - mean[c]) / std[c];
        if (out_f16) ((uint16_t*)out)[o] = oracle_f64_to_f16(yv);
        else ((float*)out)[o] = (float)yv;
      }
  free(full);
  return 0;
}

/* ------------------------------------------------------------- geometry ---
 * R4: decoded luma size ceil(W/k) x ceil(H/k); chroma ceil(W/2k) x ceil(H/2k).
 * R7: short-side resize as torchvision: short -> S, long -> floor(S*long/short);
 *     centre crop offset round((Wr-cw)/2) with round-half-to-even. */
static int32_t oracle_ceil_div(int32_t a, int32_t b) { return (a + b - 1) / b; }
static int32_t oracle_round_half_even_half(int32_t n) {   /* round(n / 2) */
  if (n % 2 == 0) return n / 2;
  int32_t lo = (n - 1) / 2;                                /* n odd, n >= 0 */
  return (lo % 2 == 0) ? lo : lo + 1;
}

int oracle_geometry_of(const oracle_params* p, int32_t width, int32_t height, oracle_geometry* g) {
  return oracle_geometry_of2(p, width, height, 2, 2, g);
}

int oracle_geometry_of2(const oracle_params* p, int32_t width, int32_t height, int32_t hs,
                        int32_t vs, oracle_geometry* g) {
  if (!p || !g || width <= 0 || height <= 0) return 1;
  int32_t k = p->scale_denom;
  if (k != 1 && k != 2 && k != 4 && k != 8) return 2;
  if ((hs != 1 && hs != 2) || (vs != 1 && vs != 2)) return 5;
  g->Wd = oracle_ceil_div(width, k);
  g->Hd = oracle_ceil_div(height, k);
  /* component size ceil(X/hs) (T.81 A.1.1), decoded at 1/k: ceil(X/(hs k)) */
  g->Wc = oracle_ceil_div(width, hs * k);
  g->Hc = oracle_ceil_div(height, vs * k);
  if (p->resize_mode == 0) {
    int32_t S = p->resize_short;
    if (S <= 0) return 3;
    if (g->Wd <= g->Hd) { g->Wr = S; g->Hr = (int32_t)(((long long)S * g->Hd) / g->Wd); }
    else                { g->Hr = S; g->Wr = (int32_t)(((long long)S * g->Wd) / g->Hd); }
  } else {
    if (p->resize_w <= 0 || p->resize_h <= 0) return 3;
    g->Wr = p->resize_w; g->Hr = p->resize_h;
  }
  if (p->crop_w > 0 || p->crop_h > 0) {
    if (p->crop_w <= 0 || p->crop_h <= 0 || p->crop_w > g->Wr || p->crop_h > g->Hr) return 4;
    g->OW = p->crop_w; g->OH = p->crop_h;
    g->left = oracle_round_half_even_half(g->Wr - p->crop_w);
    g->top = oracle_round_half_even_half(g->Hr - p->crop_h);
  } else {
    g->OW = g->Wr; g->OH = g->Hr; g->left = 0; g->top = 0;
  }
  return 0;
}

int oracle_run_image(const oracle_params* p, const oracle_image* im, int32_t left, int32_t top, void* out) {
  return oracle_run_image2(p, im, left, top, 0, 0, 0, 0, out);
}

int oracle_run_image2(const oracle_params* p, const oracle_image* im, int32_t left, int32_t top,
                      int32_t roi_x, int32_t roi_y, int32_t roi_w, int32_t roi_h, void* out) {
  oracle_geometry g;
  int32_t hs = im->comp[1].coef == NULL ? 2 : im->hs, vs = im->comp[1].coef == NULL ? 2 : im->vs;
  int rc = oracle_geometry_of2(p, im->width, im->height, hs, vs, &g);
  if (rc) return rc;
  /* reading R18 (libjpeg-turbo scaled decoding of 4:2:0): chroma blocks are
   * decoded at scale 1/(k/2), which puts chroma on the luma grid
   * (ceil(W/k) x ceil(H/k)); no upsampling follows (factors 1, 1) */
  int32_t ck = p->scale_denom;
  if (p->chroma_2s && im->comp[1].coef != NULL) {
    if (p->scale_denom < 2 || hs != 2 || vs != 2) return 22;
    ck = p->scale_denom / 2;
    g.Wc = g.Wd; g.Hc = g.Hd;
    hs = vs = 1;
  }
  if (left >= 0 && top >= 0) { g.left = left; g.top = top; }
  int32_t wx0 = 0, wy0 = 0, ww = 0, wh = 0;     /* decoded ROI window (reading R15) */
  if (roi_w > 0 || roi_h > 0) {
    const int32_t k = p->scale_denom;
    if (roi_w <= 0 || roi_h <= 0 || roi_x < 0 || roi_y < 0 || roi_x + roi_w > im->width ||
        roi_y + roi_h > im->height)
      return 20;
    wx0 = roi_x / k; wy0 = roi_y / k;
    ww = oracle_ceil_div(roi_x + roi_w, k) - wx0;
    wh = oracle_ceil_div(roi_y + roi_h, k) - wy0;
    /* output = the plan's size; the window is resized to it, no crop */
    g.OW = p->crop_w > 0 ? p->crop_w : p->resize_w;
    g.OH = p->crop_w > 0 ? p->crop_h : p->resize_h;
    if (g.OW <= 0 || g.OH <= 0) return 21;
  }
  uint8_t* Y = (uint8_t*)malloc((size_t)g.Wd * g.Hd);
  uint8_t* Cb = (uint8_t*)malloc((size_t)g.Wc * g.Hc);
  uint8_t* Cr = (uint8_t*)malloc((size_t)g.Wc * g.Hc);
  uint8_t* rgb = (uint8_t*)malloc((size_t)g.Wd * g.Hd * 3);
  rc = 10;
  if (Y && Cb && Cr && rgb) {
    rc = oracle_decode_plane2(&im->comp[0], p->scale_denom, p->idct_def, g.Wd, g.Hd, NULL, Y);
    if (im->comp[1].coef == NULL) {
      /* grayscale (one component, T.81 A.1.1 Nf = 1): the JFIF colour space
       * is Y only, i.e. R = G = B = Y (R6 with Cb = Cr = 128) */
      for (int32_t i = 0; !rc && i < g.Wd * g.Hd; ++i)
        rgb[3 * i] = rgb[3 * i + 1] = rgb[3 * i + 2] = Y[i];
    } else {
      if (!rc) rc = oracle_decode_plane2(&im->comp[1], ck, p->idct_def, g.Wc, g.Hc, NULL, Cb);
      if (!rc) rc = oracle_decode_plane2(&im->comp[2], ck, p->idct_def, g.Wc, g.Hc, NULL, Cr);
      if (!rc) rc = oracle_upsample_color2(Y, g.Wd, g.Hd, Cb, Cr, g.Wc, g.Hc, hs, vs, NULL, rgb);
    }
    if (!rc && ww > 0) {
      /* crop the decoded RGB image to the ROI window, then resize the
       * window to the output size (P:1080-1083 face crops at a fixed DNN
       * input size; reading R15) */
      uint8_t* win = (uint8_t*)malloc((size_t)ww * wh * 3);
      if (!win) rc = 11;
      for (int32_t y = 0; !rc && y < wh; ++y)
        memcpy(win + (size_t)y * ww * 3, rgb + ((size_t)(wy0 + y) * g.Wd + wx0) * 3, (size_t)ww * 3);
      if (!rc) rc = oracle_resize_crop_normalize(win, ww, wh, g.OW, g.OH, 0, 0, g.OW, g.OH, p->mean,
                                                 p->std, p->out_f16, out, NULL);
      free(win);
    } else if (!rc) {
      rc = oracle_resize_crop_normalize(rgb, g.Wd, g.Hd, g.Wr, g.Hr, g.left, g.top,
                                        g.OW, g.OH, p->mean, p->std, p->out_f16, out, NULL);
    }
  }
  free(Y); free(Cb); free(Cr); free(rgb);
  return rc;
}

/* Algorithm 1: ratio-preserving resize to short side = target,
 * l,t = (w'-target)/2, (h'-target)/2; r,b = l+target, t+target;
 * scale = min(h,w)/target; bounds multiplied by scale.  SPEC S:390-398 rounds
 * l',t' down and r',b' up. */
int oracle_alg1_crop_window(int32_t height, int32_t width, int32_t target,
                            int32_t* l, int32_t* r, int32_t* t, int32_t* b) {
  if (height <= 0 || width <= 0 || target <= 0) return 1;
  int32_t mn = height < width ? height : width;
  if (mn < target) return 2;
  double hp, wp;
  if (height <= width) { hp = target; wp = floor((double)target * width / height); }
  else                 { wp = target; hp = floor((double)target * height / width); }
  double lf = (wp - target) / 2.0, tf = (hp - target) / 2.0;
  double rf = lf + target, bf = tf + target;
  /* scale * bound, evaluated as min(h,w) * bound / target (one rounding) */
  *l = (int32_t)floor((double)mn * lf / (double)target);
  *t = (int32_t)floor((double)mn * tf / (double)target);
  *r = (int32_t)ceil((double)mn * rf / (double)target);
  *b = (int32_t)ceil((double)mn * bf / (double)target);
  return 0;
}
