/*
 * smol_oracle.h -- plain, slow CPU oracle for the Smol preprocessing hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load or call this.  It
 * shares no code, header, table or constant generator with the CUDA path
 * (paper_2007_13005_b200/csrc, include/smol_preproc.h).
 *
 * What it computes (SURVEY §8(c) "Oracle algorithm"):
 * the UNFUSED, NON-ROI pipeline of the paper's preprocessing steps
 *   1. decode (§6.4 "entropy decoding, inverse transform,
 *      post-processing"; entropy decoding done by the host):
 *      dequantize + 8x8 IDCT (ITU-T T.81 A.3.3) at scale 1, or the k x k box
 *      mean of it at scale 1/k (reading R1; Definition B, R16, as an
 *      option) + level shift, round half up, clamp to u8 (R3);  centred
 *      triangle chroma upsample per subsampled axis (4:2:0, 4:2:2; 4:4:4
 *      needs none) (R2);
 *      exact JFIF YCbCr->RGB (R6);
 *   2. resize (short edge -> S, or exact) with half-pixel bilinear, no
 *      antialias (readings R7/R8), centre crop (R7);
 *   3. convert to float, /255, -mean, /std;
 *   4. channels-first.
 * All floating point is IEEE double; integer steps are exact.
 *
 * Every function returns 0 on success, nonzero on invalid arguments.
 */
#ifndef SMOL_ORACLE_H
#define SMOL_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* One component's coefficient plane: [blocks_h][blocks_w][64] int16 in
 * natural (row-major v*8+u) order, absolute DC; row stride in ELEMENTS.
 * q: 64-entry natural-order quantization table. */
typedef struct {
  const int16_t* coef;
  int32_t blocks_w, blocks_h, row_stride;
  const uint16_t* q;
} oracle_plane;

typedef struct {
  int32_t width, height;      /* SOF size in pixels */
  oracle_plane comp[3];       /* Y, Cb, Cr; comp[1].coef == NULL: grayscale
                                 (one component; R = G = B = Y) */
  int32_t hs, vs;             /* chroma subsampling factors (T.81 A.1.1: Hmax/Hc,
                                 Vmax/Vc): 2,2 = 4:2:0; 2,1 = 4:2:2; 1,1 = 4:4:4 */
} oracle_image;

typedef struct {
  int32_t scale_denom;        /* k in {1,2,4,8}: decode at scale 1/k */
  int32_t resize_mode;        /* 0 = short side -> resize_short, 1 = exact */
  int32_t resize_short, resize_w, resize_h;
  int32_t crop_w, crop_h;     /* 0,0 = no crop */
  double mean[3], std[3];
  int32_t out_f16;            /* 0 = fp32 output, 1 = fp16 (RNE) */
  int32_t idct_def;           /* reduced-scale IDCT: 0 = Definition A (box mean,
                                 reading R1), 1 = Definition B (truncated
                                 (8/k)-point IDCT, reading R16) */
  int32_t chroma_2s;          /* 1 (k >= 2, 4:2:0): chroma decoded at scale
                                 1/(k/2), i.e. at the luma resolution, and used
                                 without upsampling (reading R18) */
} oracle_params;

typedef struct {
  int32_t Wd, Hd;             /* decoded luma size at scale 1/k */
  int32_t Wc, Hc;             /* decoded chroma size */
  int32_t Wr, Hr;             /* resized size */
  int32_t left, top;          /* crop offset in resized coordinates */
  int32_t OW, OH;             /* output size */
} oracle_geometry;

/* Geometry per readings R4 (decoded sizes), R7 (torchvision resize/crop),
 * 4:2:0 chroma. */
int oracle_geometry_of(const oracle_params* p, int32_t width, int32_t height,
                       oracle_geometry* g);
/* Same for chroma subsampled by hs x vs (T.81 A.1.1: component size
 * ceil(X / hs) x ceil(Y / vs), then ceil(./k) at scale 1/k, reading R4). */
int oracle_geometry_of2(const oracle_params* p, int32_t width, int32_t height, int32_t hs,
                        int32_t vs, oracle_geometry* g);

/* Decode one component at scale 1/k into an out_w x out_h plane.
 * v_out (nullable): unrounded IDCT value before the +128 level shift.
 * u8_out: clamp(floor(v + 128 + 1/2), 0, 255). */
int oracle_decode_plane(const oracle_plane* pl, int32_t k, int32_t out_w, int32_t out_h,
                        double* v_out, uint8_t* u8_out);
/* Same with the reduced-scale definition idct_def (0: A, box mean; 1: B,
 * truncated (8/k)-point IDCT of the top-left (8/k)^2 coefficients). */
int oracle_decode_plane2(const oracle_plane* pl, int32_t k, int32_t idct_def, int32_t out_w,
                         int32_t out_h, double* v_out, uint8_t* u8_out);

/* 4:2:0 upsample + YCbCr->RGB.  Y: [Hd][Wd]; Cb, Cr: [Hc][Wc].
 * c16_out (nullable): [Hd][Wd][2] upsampled Cb, Cr in 1/16 units.
 * rgb_out: [Hd][Wd][3]. */
int oracle_upsample_color(const uint8_t* Y, int32_t Wd, int32_t Hd,
                          const uint8_t* Cb, const uint8_t* Cr, int32_t Wc, int32_t Hc,
                          int32_t* c16_out, uint8_t* rgb_out);

/* Upsample (hs x vs subsampled chroma; reading R2 per axis: factor 2 = the
 * centred triangle 3/4, 1/4, factor 1 = identity) + YCbCr->RGB. */
int oracle_upsample_color2(const uint8_t* Y, int32_t Wd, int32_t Hd,
                           const uint8_t* Cb, const uint8_t* Cr, int32_t Wc, int32_t Hc,
                           int32_t hs, int32_t vs, int32_t* c16_out, uint8_t* rgb_out);

/* JFIF colour conversion of one sample, chroma in 1/16 units (0..4080). */
void oracle_color(int32_t Y, int32_t cb16, int32_t cr16, uint8_t rgb[3]);

/* Bilinear resize of the whole [Hd][Wd][3] image to Wr x Hr, crop the
 * OW x OH window at (left, top), normalize, write [3][OH][OW] (f32 or f16
 * bits).  resized_out (nullable): [3][OH][OW] doubles before normalization. */
int oracle_resize_crop_normalize(const uint8_t* rgb, int32_t Wd, int32_t Hd,
                                 int32_t Wr, int32_t Hr, int32_t left, int32_t top,
                                 int32_t OW, int32_t OH, const double mean[3],
                                 const double std[3], int32_t out_f16, void* out,
                                 double* resized_out);

/* Whole pipeline for one image.  left/top < 0 = centre crop (R7); otherwise
 * an explicit crop offset in resized coordinates (the optional ROI,
 * P:1107-1109).  out: [3][OH][OW]. */
int oracle_run_image(const oracle_params* p, const oracle_image* im,
                     int32_t left, int32_t top, void* out);

/* Whole pipeline with an optional ROI rectangle (P:1080-1083, P:1107-1109:
 * "the ROIs are the face crops"; reading R15): roi_w, roi_h > 0 select the
 * SOF-pixel rectangle [roi_x, roi_x + roi_w) x [roi_y, roi_y + roi_h); its
 * decoded window at scale 1/k is [floor(x/k), ceil((x+w)/k)) x likewise;
 * the decoded RGB image is cropped to that window, which is resized to the
 * plan's output size (crop_w x crop_h, else resize_w x resize_h) -- crop,
 * then resize (torchvision resized_crop); normalize; channels-first.
 * roi_w = roi_h = 0: oracle_run_image(p, im, left, top, out). */
int oracle_run_image2(const oracle_params* p, const oracle_image* im, int32_t left, int32_t top,
                      int32_t roi_x, int32_t roi_y, int32_t roi_w, int32_t roi_h, void* out);

/* Algorithm 1 crop window in source coordinates, SPEC
 * convention: l',t' floored, r',b' ceiled.  Geometry helper only
 * (reading R12); not used for sampling. */
int oracle_alg1_crop_window(int32_t height, int32_t width, int32_t target,
                            int32_t* l, int32_t* r, int32_t* t, int32_t* b);

/* Round a double to IEEE binary16 (round to nearest even); returns bits. */
uint16_t oracle_f64_to_f16(double x);

/* ---- baseline JPEG entropy decoding (smol_oracle_jpeg.c)
 * ITU-T T.81 Annexes B, C, F.2.2 followed sequentially (see that file).
 * Accepts one baseline (SOF0/SOF1, 8-bit, Huffman) interleaved scan of 1 or
 * 3 components, with or without restart intervals. */
typedef struct {
  int32_t width, height, ncomp;
  int32_t h[3], v[3];            /* sampling factors (SOF) */
  int32_t tq[3];                 /* quantization table selectors */
  int32_t blocks_w[3], blocks_h[3];   /* coefficient blocks per component incl.
                                         MCU padding (A.2.2 / A.2.3) */
  int32_t mcus_x, mcus_y;
  int32_t restart_interval;      /* MCUs per restart interval (DRI), 0 = none */
  uint16_t qt[4][64];            /* DQT tables, natural order */
} oracle_jpeg_info;

/* Header of a JPEG file (0 = ok; nonzero = not a supported baseline file). */
int oracle_jpeg_info_of(const uint8_t* data, int64_t size, oracle_jpeg_info* info);
/* Entropy-decode the scan into planes[c]: [blocks_h][blocks_w][64] int16,
 * natural order, absolute DC (caller-allocated, sizes from the info). */
int oracle_jpeg_decode(const uint8_t* data, int64_t size, int16_t* const planes[3]);

#ifdef __cplusplus
}
#endif
#endif
