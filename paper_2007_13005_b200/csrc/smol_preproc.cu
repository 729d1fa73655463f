// smol_preproc.cu -- host runtime of the C ABI declared in
// include/smol_preproc.h: parameter/descriptor validation, per-image
// geometry, device descriptor upload (pinned ring, no allocation per run),
// kernel selection per (scale, dtype) and launch.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <algorithm>
#include <array>
#include <climits>
#include <mutex>
#include <new>
#include <string>
#include <vector>

#include "smol_preproc.h"
#include "smol_geom.cuh"
#include "smol_kernels.cuh"
#include "smol_compact.cuh"
#include "smol_thumb.cuh"
#include "smol_jpeg.cuh"
#include "smol_launch.h"

using namespace smol;

namespace {

thread_local std::string g_last_error;

int32_t fail(int32_t code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_last_error = buf;
  return code;
}

#define SMOL_CUDA(call)                                                             \
  do {                                                                              \
    cudaError_t e_ = (call);                                                        \
    if (e_ != cudaSuccess)                                                          \
      return fail(SMOL_ERR_CUDA, "%s: %s (%s:%d)", #call, cudaGetErrorString(e_),  \
                  __FILE__, __LINE__);                                              \
  } while (0)

constexpr int kRing = 4;           // descriptor ring depth (runs in flight per plan)
constexpr int kStageMax = 4, kStageDefault = 3;   // staging slots of the staged paths (SMOL_STAGE_SLOTS)
constexpr int kTapCap = 8192;      // int4 words of host-computed taps per run (128 KB; the rest: per CTA)
constexpr int kMaxDevices = 64;

// ------------------------------------------------------------ basis upload --
// Definitions in smol_kernels.cuh (struct Basis); reading R1.
void init_basis(Basis& b) {
  const double pi = 3.14159265358979323846;
  double t[8][8];
  for (int u = 0; u < 8; ++u)
    for (int x = 0; x < 8; ++x) {
      if (u == 0) t[u][x] = 1.0;
      else if (u == 4) t[u][x] = ((2 * x + 1) % 8 == 1 || (2 * x + 1) % 8 == 7) ? 1.0 : -1.0;
      else t[u][x] = std::sqrt(2.0) * std::cos((2 * x + 1) * u * pi / 16.0);
    }
  for (int u = 0; u < 8; ++u)
    for (int x = 0; x < 4; ++x) b.t[u][x] = (float)t[u][x];
  // box means; entries that vanish by the sum-of-cosines identity are exact 0
  auto box = [&](int k, int u, int j) -> double {
    if (u > 0 && ((k * u) % 16 == 0 || (k * u * (2 * j + 1)) % 16 == 8)) return 0.0;
    double s = 0;
    for (int x = j * k; x < j * k + k; ++x) s += t[u][x];
    return s / k;
  };
  for (int k = 0; k < 4; ++k)
    for (int y = 0; y < 4; ++y) b.tp[k][y] = make_float2((float)t[2 * k][y], (float)t[2 * k + 1][y]);
  for (int j = 0; j < 2; ++j)
    for (int u = 0; u < 8; ++u) b.a2[j][u] = (float)box(2, u, j);
  for (int u = 0; u < 8; ++u) b.a4[u] = (float)box(4, u, 0);
  // JFIF R and B (reading R6) in fp32; the exhaustive check of these exact
  // recipes is tests/test_color_fp32.py
  b.kR = (float)(1.402 / 16.0);
  b.kB = (float)(1.772 / 16.0);
  b.cR = (float)(0.5 - 2048.0 * 1.402 / 16.0);
  b.cB = (float)(0.5 - 2048.0 * 1.772 / 16.0 + 1.0 / 8192.0);
  b.gK1 = 543917632u;
  b.gCb = (uint32_t)-43017;
  b.gCr = (uint32_t)-89267;
}

std::mutex g_basis_mu;
bool g_basis_done[kMaxDevices] = {};

int32_t ensure_basis(int dev) {
  std::lock_guard<std::mutex> lk(g_basis_mu);
  if (dev < 0 || dev >= kMaxDevices) return fail(SMOL_ERR_CUDA, "device index %d out of range", dev);
  if (g_basis_done[dev]) return SMOL_OK;
  Basis b;
  init_basis(b);
  SMOL_CUDA(cudaMemcpyToSymbol(c_basis, &b, sizeof(Basis)));     // this unit (thumbnail kernel)
  SMOL_CUDA(upload_basis_k1(b));
  SMOL_CUDA(upload_basis_k2(b));
  SMOL_CUDA(upload_basis_k4(b));
  SMOL_CUDA(upload_basis_k8(b));
  g_basis_done[dev] = true;
  return SMOL_OK;
}

// ------------------------------------------------------------- validation --
int32_t validate_params(const smol_preproc_params* p) {
  if (!p) return fail(SMOL_ERR_INVALID, "params is NULL");
  if (p->scale_denom != 1 && p->scale_denom != 2 && p->scale_denom != 4 && p->scale_denom != 8)
    return fail(SMOL_ERR_INVALID, "params.scale_denom=%d not in {1,2,4,8}", p->scale_denom);
  if (p->resize_mode == SMOL_RESIZE_SHORT_SIDE) {
    if (p->resize_short <= 0) return fail(SMOL_ERR_INVALID, "params.resize_short=%d <= 0", p->resize_short);
    if (p->crop_w <= 0 || p->crop_h <= 0)
      return fail(SMOL_ERR_INVALID, "SHORT_SIDE resize needs crop_w, crop_h > 0 (fixed output size)");
  } else if (p->resize_mode == SMOL_RESIZE_EXACT) {
    if (p->resize_w <= 0 || p->resize_h <= 0)
      return fail(SMOL_ERR_INVALID, "params.resize_w/h=%d/%d must be > 0", p->resize_w, p->resize_h);
    if ((p->crop_w > 0) != (p->crop_h > 0) || p->crop_w < 0 || p->crop_h < 0)
      return fail(SMOL_ERR_INVALID, "params.crop_w/h=%d/%d: both > 0 or both 0", p->crop_w, p->crop_h);
    if (p->crop_w > p->resize_w || p->crop_h > p->resize_h)
      return fail(SMOL_ERR_INVALID, "crop %dx%d larger than resize %dx%d", p->crop_w, p->crop_h,
                  p->resize_w, p->resize_h);
  } else {
    return fail(SMOL_ERR_INVALID, "params.resize_mode=%d", p->resize_mode);
  }
  for (int c = 0; c < 3; ++c) {
    if (!(p->std[c] > 0.f) || !std::isfinite(p->std[c]) || !std::isfinite(p->mean[c]))
      return fail(SMOL_ERR_INVALID, "params.std[%d]=%g must be finite and > 0", c, (double)p->std[c]);
  }
  if (p->out_dtype != SMOL_OUT_F32_NCHW && p->out_dtype != SMOL_OUT_F16_NCHW)
    return fail(SMOL_ERR_INVALID, "params.out_dtype=%d", p->out_dtype);
  if (p->layout != SMOL_LAYOUT_DENSE64 && p->layout != SMOL_LAYOUT_PACKED)
    return fail(SMOL_ERR_INVALID, "params.layout=%d", p->layout);
  if (p->tile_rows < 0 || p->tile_rows > 4096)
    return fail(SMOL_ERR_INVALID, "params.tile_rows=%d", p->tile_rows);
  if (p->idct_def != SMOL_IDCT_BOX_MEAN && p->idct_def != SMOL_IDCT_TRUNCATED)
    return fail(SMOL_ERR_INVALID, "params.idct_def=%d", p->idct_def);
  if (p->chroma_2s != 0 && p->chroma_2s != 1)
    return fail(SMOL_ERR_INVALID, "params.chroma_2s=%d", p->chroma_2s);
  if (p->chroma_2s && (p->scale_denom < 2 || p->layout != SMOL_LAYOUT_DENSE64 || p->idct_def != SMOL_IDCT_BOX_MEAN))
    return fail(SMOL_ERR_UNSUPPORTED, "params.chroma_2s needs scale_denom >= 2, the DENSE64 layout and "
                "Definition A");
  if (p->max_width < 0 || p->max_height < 0 || (p->max_width > 0) != (p->max_height > 0) ||
      p->max_width > 65535 || p->max_height > 65535)
    return fail(SMOL_ERR_INVALID, "params.max_width/max_height=%d/%d: both in [1, 65535] or both 0",
                p->max_width, p->max_height);
  return SMOL_OK;
}

// coefficients per block the scale uses: Definition A (reading R1: the
// box-averaged basis of the others is exactly zero) 64 / 49 / 25 / 1 at 1,
// 1/2, 1/4, 1/8; Definition B (R16) the top-left (8/k)^2: 64 / 16 / 4 / 1
int used_coefs(int K, int def) {
  if (def == SMOL_IDCT_TRUNCATED) return (8 / K) * (8 / K);
  return K == 1 ? 64 : K == 2 ? 49 : K == 4 ? 25 : 1;
}

// int16 elements per coefficient block of a layout at scale 1/K
// (smol_kernels.cuh BlockFmt)
int block_elems(int K, int layout, int def) {
  if (layout != SMOL_LAYOUT_PACKED || K == 1) return 64;
  if (def == SMOL_IDCT_TRUNCATED) return (8 / K) * (8 / K);
  return K == 2 ? 52 : K == 4 ? 28 : 1;
}

// ---- JPEG headers (T.81 Annex B) ----------------------
constexpr int kMaxJpegQt = 64, kMaxHuffSets = 16;

// Figure A.6 zig-zag order: position k -> natural index, built by walking
// the anti-diagonals (even ones upwards).
std::array<int, 64> zigzag_order() {
  std::array<int, 64> z{};
  int k = 0;
  for (int s = 0; s < 15; ++s)
    for (int i = 0; i < 8; ++i) {
      const int v = (s % 2 == 0) ? std::min(s, 7) - i : std::max(0, s - 7) + i;   // row
      const int u = s - v;
      if (v < 0 || v > 7 || u < 0 || u > 7) continue;
      z[k++] = v * 8 + u;
    }
  return z;
}

struct JpegHdr {
  int32_t width = 0, height = 0, ncomp = 0, subsampling = 0;
  int32_t h[3] = {}, v[3] = {}, tq[3] = {}, td[3] = {}, ta[3] = {};
  int32_t ri = 0, scan_off = 0, mcus_x = 0, mcus_y = 0, nseg = 0;
  int32_t blocks_w[3] = {}, blocks_h[3] = {};
  uint16_t qt[4][64] = {};
  bool qt_ok[4] = {};
  // DHT contents per (class, id): BITS, HUFFVAL (kept raw for the table-set dedupe)
  uint8_t bits[2][4][16] = {};
  uint8_t vals[2][4][256] = {};
  bool ht_ok[2][4] = {};
};

unsigned be16(const uint8_t* p) { return ((unsigned)p[0] << 8) | p[1]; }

// T.81 Annex C code assignment (canonical: codes of one length consecutive,
// next length = (last + 1) << 1); false if the counts overflow a prefix code.
bool huff_valid(const uint8_t* bits) {
  long long code = 0;
  for (int l = 1; l <= 16; ++l) {
    code += bits[l - 1];
    if (code > (1LL << l)) return false;
    code <<= 1;
  }
  return true;
}

void build_huff(const uint8_t* bits, const uint8_t* vals, HuffTable& t) {
  memset(&t, 0, sizeof(t));
  int code = 0, j = 0;
  for (int l = 1; l <= 16; ++l) {
    const int n = bits[l - 1];
    t.valoff[l] = j - code;                     // HUFFVAL index = code + valoff (F.15: VALPTR - MINCODE)
    for (int i = 0; i < n; ++i, ++code, ++j)
      if (l <= kHuffLutBits)
        for (int f = code << (kHuffLutBits - l); f < (code + 1) << (kHuffLutBits - l); ++f)
          t.lut[f] = (uint16_t)(l << 8 | vals[j]);
    t.limit[l] = (uint32_t)code << (16 - l);    // first code of length > l, left-justified
    code <<= 1;
  }
  memcpy(t.huffval, vals, 256);
}

// Decoder tables of an absent (never referenced) table: every window invalid.
void empty_huff(HuffTable& t) {
  memset(&t, 0, sizeof(t));
}

// Header of one file; on error a status + message naming image idx.
int32_t parse_jpeg(const uint8_t* d, int64_t size, int idx, JpegHdr& H) {
  H = JpegHdr{};
  static const std::array<int, 64> zz = zigzag_order();
  if (size < 4 || d[0] != 0xFF || d[1] != 0xD8) return fail(SMOL_ERR_INVALID, "image %d: no SOI marker", idx);
  int64_t i = 2;
  bool sof = false;
  while (true) {
    if (i + 4 > size) return fail(SMOL_ERR_INVALID, "image %d: header runs past the file end", idx);
    if (d[i] != 0xFF) return fail(SMOL_ERR_INVALID, "image %d: marker expected at byte %lld", idx, (long long)i);
    const unsigned m = d[i + 1];
    if (m == 0xFF) { ++i; continue; }
    const unsigned len = be16(d + i + 2);
    if (len < 2 || i + 2 + len > size) return fail(SMOL_ERR_INVALID, "image %d: segment length at byte %lld", idx, (long long)i);
    const uint8_t* p = d + i + 4;
    const int plen = (int)len - 2;
    if (m == 0xDB) {                                               // DQT (B.2.4.1)
      for (int o = 0; o < plen;) {
        const int pq = p[o] >> 4, t = p[o] & 15;
        if (pq != 0) return fail(SMOL_ERR_UNSUPPORTED, "image %d: 16-bit quantization table", idx);
        if (t > 3 || o + 65 > plen) return fail(SMOL_ERR_INVALID, "image %d: bad DQT", idx);
        for (int k = 0; k < 64; ++k) H.qt[t][zz[k]] = p[o + 1 + k];
        H.qt_ok[t] = true;
        o += 65;
      }
    } else if (m == 0xC4) {                                        // DHT (B.2.4.2)
      for (int o = 0; o < plen;) {
        if (o + 17 > plen) return fail(SMOL_ERR_INVALID, "image %d: bad DHT", idx);
        const int tc = p[o] >> 4, th = p[o] & 15;
        int nv = 0;
        for (int k = 0; k < 16; ++k) nv += p[o + 1 + k];
        if (tc > 1 || th > 3 || nv > 256 || o + 17 + nv > plen || !huff_valid(p + o + 1))
          return fail(SMOL_ERR_INVALID, "image %d: bad DHT", idx);
        memcpy(H.bits[tc][th], p + o + 1, 16);
        memset(H.vals[tc][th], 0, 256);
        memcpy(H.vals[tc][th], p + o + 17, (size_t)nv);
        H.ht_ok[tc][th] = true;
        o += 17 + nv;
      }
    } else if (m == 0xC0 || m == 0xC1) {                           // SOF0/1 (B.2.2)
      if (plen < 6) return fail(SMOL_ERR_INVALID, "image %d: bad SOF", idx);
      if (p[0] != 8) return fail(SMOL_ERR_UNSUPPORTED, "image %d: %d-bit samples", idx, p[0]);
      H.height = (int32_t)be16(p + 1);
      H.width = (int32_t)be16(p + 3);
      H.ncomp = p[5];
      if ((H.ncomp != 1 && H.ncomp != 3) || plen < 6 + 3 * H.ncomp)
        return fail(SMOL_ERR_UNSUPPORTED, "image %d: %d components", idx, H.ncomp);
      if (H.width <= 0 || H.height <= 0) return fail(SMOL_ERR_INVALID, "image %d: zero size (DNL)", idx);
      for (int c = 0; c < H.ncomp; ++c) {
        H.h[c] = p[7 + 3 * c] >> 4;
        H.v[c] = p[7 + 3 * c] & 15;
        H.tq[c] = p[8 + 3 * c];
        if (H.tq[c] > 3) return fail(SMOL_ERR_INVALID, "image %d: bad Tq", idx);
      }
      sof = true;
    } else if (m >= 0xC2 && m <= 0xCF && m != 0xC4 && m != 0xC8 && m != 0xCC) {
      return fail(SMOL_ERR_UNSUPPORTED, "image %d: not baseline sequential Huffman (SOF 0x%02X)", idx, m);
    } else if (m == 0xDD) {                                        // DRI (B.2.4.4)
      if (plen < 2) return fail(SMOL_ERR_INVALID, "image %d: bad DRI", idx);
      H.ri = (int32_t)be16(p);
    } else if (m == 0xDA) {                                        // SOS (B.2.3)
      if (!sof || plen < 1) return fail(SMOL_ERR_INVALID, "image %d: SOS before SOF", idx);
      const int ns = p[0];
      if (ns != H.ncomp || plen < 1 + 2 * ns + 3)
        return fail(SMOL_ERR_UNSUPPORTED, "image %d: scan of %d of %d components", idx, ns, H.ncomp);
      for (int j = 0; j < ns; ++j) {
        H.td[j] = p[2 + 2 * j] >> 4;
        H.ta[j] = p[2 + 2 * j] & 15;
        if (H.td[j] > 3 || H.ta[j] > 3 || !H.ht_ok[0][H.td[j]] || !H.ht_ok[1][H.ta[j]])
          return fail(SMOL_ERR_INVALID, "image %d: scan uses an undefined Huffman table", idx);
      }
      if (p[1 + 2 * ns] != 0 || p[2 + 2 * ns] != 63 || p[3 + 2 * ns] != 0)
        return fail(SMOL_ERR_UNSUPPORTED, "image %d: not a baseline scan (Ss/Se/Ah/Al)", idx);
      if (i + 2 + len > INT_MAX || size > INT_MAX) return fail(SMOL_ERR_UNSUPPORTED, "image %d: file >= 2 GiB", idx);
      H.scan_off = (int32_t)(i + 2 + len);
      break;
    }
    i += 2 + len;
  }
  for (int c = 0; c < H.ncomp; ++c)
    if (!H.qt_ok[H.tq[c]]) return fail(SMOL_ERR_INVALID, "image %d: undefined quantization table", idx);
  if (H.ncomp == 1) {
    H.subsampling = 400;
    H.blocks_w[0] = ceil_div(H.width, 8);                          // A.2.2: non-interleaved
    H.blocks_h[0] = ceil_div(H.height, 8);
    H.mcus_x = H.blocks_w[0];
    H.mcus_y = H.blocks_h[0];
  } else {
    if (H.h[1] != 1 || H.v[1] != 1 || H.h[2] != 1 || H.v[2] != 1)
      return fail(SMOL_ERR_UNSUPPORTED, "image %d: chroma sampling factors must be 1x1", idx);
    if (H.h[0] == 2 && H.v[0] == 2) H.subsampling = 420;
    else if (H.h[0] == 2 && H.v[0] == 1) H.subsampling = 422;
    else if (H.h[0] == 1 && H.v[0] == 1) H.subsampling = 444;
    else return fail(SMOL_ERR_UNSUPPORTED, "image %d: luma sampling %dx%d", idx, H.h[0], H.v[0]);
    H.mcus_x = ceil_div(H.width, 8 * H.h[0]);                     // A.2.3: interleaved
    H.mcus_y = ceil_div(H.height, 8 * H.v[0]);
    for (int c = 0; c < 3; ++c) { H.blocks_w[c] = H.mcus_x * H.h[c]; H.blocks_h[c] = H.mcus_y * H.v[c]; }
  }
  const long long nmcu = (long long)H.mcus_x * H.mcus_y;
  H.nseg = H.ri > 0 ? (int32_t)((nmcu + H.ri - 1) / H.ri) : 1;
  return SMOL_OK;
}

// Per-image geometry (readings R4, R7, R11); fills the device descriptor's
// size fields.  idx is the image index for error messages.
int32_t image_geometry(const smol_preproc_params* p, const smol_image_desc* d, int idx, DevImage& g) {
  const int k = p->scale_denom;
  if (d->width <= 0 || d->height <= 0)
    return fail(SMOL_ERR_INVALID, "image %d: width/height=%d/%d must be > 0", idx, d->width, d->height);
  if (d->width > 65535 || d->height > 65535)
    return fail(SMOL_ERR_INVALID, "image %d: width/height=%d/%d > 65535 (JPEG limit)", idx, d->width, d->height);
  if (d->subsampling != 420 && d->subsampling != 400 && d->subsampling != 422 && d->subsampling != 444)
    return fail(SMOL_ERR_UNSUPPORTED, "image %d: subsampling=%d (420, 422, 444 or 400)", idx, d->subsampling);
  g.gray = d->subsampling == 400;
  g.hs = d->subsampling == 444 ? 1 : 2;      // T.81 A.1.1: Hmax / H_chroma, Vmax / V_chroma
  g.vs = (d->subsampling == 444 || d->subsampling == 422) ? 1 : 2;
  g.ck = k;
  g.Wd = ceil_div(d->width, k);
  g.Hd = ceil_div(d->height, k);
  g.Wc = ceil_div(d->width, g.hs * k);      // chroma ceil(W/hs) decoded at 1/k (R4)
  g.Hc = ceil_div(d->height, g.vs * k);
  if (p->chroma_2s && d->subsampling == 420) {
    // reading R18: chroma blocks decoded at 1/(k/2) -> chroma at the luma
    // size ceil(W/k) x ceil(H/k), used without upsampling (factors 1, 1)
    g.ck = k / 2;
    g.hs = g.vs = 1;
    g.Wc = g.Wd; g.Hc = g.Hd;
  } else if (p->chroma_2s && (d->subsampling == 422 || d->subsampling == 444)) {
    return fail(SMOL_ERR_UNSUPPORTED, "image %d: chroma_2s is defined for 4:2:0 only", idx);
  }
  int OW, OH;
  if (p->resize_mode == SMOL_RESIZE_SHORT_SIDE) {
    const long long S = p->resize_short;
    if (g.Wd <= g.Hd) { g.Wr = (int)S; g.Hr = (int)(S * g.Hd / g.Wd); }
    else              { g.Hr = (int)S; g.Wr = (int)(S * g.Wd / g.Hd); }
  } else {
    g.Wr = p->resize_w; g.Hr = p->resize_h;
  }
  if (p->crop_w > 0) { OW = p->crop_w; OH = p->crop_h; } else { OW = g.Wr; OH = g.Hr; }
  g.sx0 = 0; g.sy0 = 0; g.sw = g.Wd; g.sh = g.Hd;
  if (d->roi_w != 0 || d->roi_h != 0 || d->roi_x != 0 || d->roi_y != 0) {
    // ROI rectangle (reading R15): its decoded
    // window [floor(x/k), ceil((x+w)/k)) x [floor(y/k), ceil((y+h)/k)) is
    // resized straight to the plan's output size (no crop)
    if (d->roi_w <= 0 || d->roi_h <= 0 || d->roi_x < 0 || d->roi_y < 0 ||
        (long long)d->roi_x + d->roi_w > d->width || (long long)d->roi_y + d->roi_h > d->height)
      return fail(SMOL_ERR_INVALID, "image %d: ROI rectangle (%d,%d,%d,%d) outside the %dx%d image", idx,
                  d->roi_x, d->roi_y, d->roi_w, d->roi_h, d->width, d->height);
    if (d->roi_left >= 0 || d->roi_top >= 0)
      return fail(SMOL_ERR_INVALID, "image %d: ROI rectangle and crop origin both given", idx);
    const int plan_ow = p->crop_w > 0 ? p->crop_w : p->resize_w;
    const int plan_oh = p->crop_w > 0 ? p->crop_h : p->resize_h;
    g.sx0 = d->roi_x / k;
    g.sy0 = d->roi_y / k;
    g.sw = ceil_div(d->roi_x + d->roi_w, k) - g.sx0;
    g.sh = ceil_div(d->roi_y + d->roi_h, k) - g.sy0;
    g.Wr = plan_ow; g.Hr = plan_oh;
    g.left = 0; g.top = 0;
    return SMOL_OK;
  }
  if (OW > g.Wr || OH > g.Hr)
    return fail(SMOL_ERR_INVALID, "image %d: crop %dx%d larger than resized %dx%d", idx, OW, OH, g.Wr, g.Hr);
  if (d->roi_left < 0 && d->roi_top < 0) {
    // torchvision centre crop: round((Wr - cw) / 2) with round-half-to-even
    auto half_even = [](int v) { return (v % 2 == 0) ? v / 2 : (((v - 1) / 2) % 2 == 0 ? (v - 1) / 2 : (v + 1) / 2); };
    g.left = half_even(g.Wr - OW);
    g.top = half_even(g.Hr - OH);
  } else {
    if (d->roi_left < 0 || d->roi_top < 0 || d->roi_left + OW > g.Wr || d->roi_top + OH > g.Hr)
      return fail(SMOL_ERR_INVALID, "image %d: roi origin (%d,%d) + %dx%d outside resized %dx%d", idx,
                  d->roi_left, d->roi_top, OW, OH, g.Wr, g.Hr);
    g.left = d->roi_left;
    g.top = d->roi_top;
  }
  return SMOL_OK;
}

// Same geometry as the previous image of the batch (its size fields can be
// reused: batches are mostly runs of equal-size images).
inline bool same_geometry(const smol_image_desc* a, const smol_image_desc* b) {
  return a->width == b->width && a->height == b->height && a->subsampling == b->subsampling &&
         a->roi_left == b->roi_left && a->roi_top == b->roi_top && a->roi_x == b->roi_x &&
         a->roi_y == b->roi_y && a->roi_w == b->roi_w && a->roi_h == b->roi_h;
}
inline void copy_geometry(const DevImage& from, DevImage& g) {
  g.Wd = from.Wd; g.Hd = from.Hd; g.Wc = from.Wc; g.Hc = from.Hc;
  g.Wr = from.Wr; g.Hr = from.Hr; g.left = from.left; g.top = from.top;
  g.gray = from.gray;
  g.sx0 = from.sx0; g.sy0 = from.sy0; g.sw = from.sw; g.sh = from.sh;
  g.hs = from.hs; g.vs = from.vs; g.ck = from.ck;
}
inline bool same_layout_inputs(const DevImage& a, const DevImage& b) {
  return a.Wd == b.Wd && a.Hd == b.Hd && a.Wc == b.Wc && a.Hc == b.Hc && a.Wr == b.Wr && a.Hr == b.Hr &&
         a.left == b.left && a.top == b.top && a.nbw[0] == b.nbw[0] && a.nbw[1] == b.nbw[1] &&
         a.gray == b.gray && a.sx0 == b.sx0 && a.sy0 == b.sy0 && a.sw == b.sw && a.sh == b.sh &&
         a.hs == b.hs && a.vs == b.vs && a.ck == b.ck;
}

int32_t validate_image(const smol_preproc_params* p, const smol_image_desc* d, int idx, int n_qtables,
                       DevImage& g, bool need_align = true, const DevImage* geom = nullptr) {
  int32_t rc = SMOL_OK;
  if (geom) copy_geometry(*geom, g);
  else rc = image_geometry(p, d, idx, g);
  if (rc) return rc;
  // block counts of the coded planes (the coded sampling, whatever scale
  // the chroma is decoded at)
  const int hsc = d->subsampling == 444 ? 1 : 2, vsc = (d->subsampling == 420 || d->subsampling == 400) ? 2 : 1;
  const int need_w[3] = {ceil_div(d->width, 8), ceil_div(d->width, 8 * hsc), ceil_div(d->width, 8 * hsc)};
  const int need_h[3] = {ceil_div(d->height, 8), ceil_div(d->height, 8 * vsc), ceil_div(d->height, 8 * vsc)};
  static const char* names[3] = {"Y", "Cb", "Cr"};
  for (int c = 0; c < 3; ++c) {
    g.nbw[c] = need_w[c];
    if (c > 0 && g.gray) {             // grayscale: chroma fields are ignored
      g.coef[c] = nullptr; g.stride[c] = 0; g.qidx[c] = 0;
      continue;
    }
    if (!d->coef[c]) return fail(SMOL_ERR_INVALID, "image %d: coef[%d] (%s) is NULL", idx, c, names[c]);
    if (need_align && reinterpret_cast<uintptr_t>(d->coef[c]) % 16)
      return fail(SMOL_ERR_INVALID, "image %d: coef[%d] not 16-byte aligned", idx, c);
    if (d->blocks_w[c] < need_w[c] || d->blocks_h[c] < need_h[c])
      return fail(SMOL_ERR_INVALID, "image %d: blocks_w[%d]=%d / blocks_h[%d]=%d < required %d / %d", idx, c,
                  d->blocks_w[c], c, d->blocks_h[c], need_w[c], need_h[c]);
    const int bb = 2 * block_elems(p->scale_denom, p->layout, p->idct_def);
    if (d->row_stride_bytes[c] < d->blocks_w[c] * bb || d->row_stride_bytes[c] % 16)
      return fail(SMOL_ERR_INVALID, "image %d: row_stride_bytes[%d]=%d (need >= %d, multiple of 16)", idx, c,
                  d->row_stride_bytes[c], d->blocks_w[c] * bb);
    if (d->qtable[c] < 0 || d->qtable[c] >= n_qtables)
      return fail(SMOL_ERR_INVALID, "image %d: qtable[%d]=%d not in [0,%d)", idx, c, d->qtable[c], n_qtables);
    g.coef[c] = d->coef[c];
    g.stride[c] = d->row_stride_bytes[c] / 2;
    g.qidx[c] = d->qtable[c];
    g.nbw[c] = need_w[c];
  }
  return SMOL_OK;
}

// Tiles per image t: every extra row tile re-decodes the MCU rows its
// footprint shares with a neighbour (~10 % more decode work per tile), while
// n*t CTAs run in ceil(n*t / slots) waves of the resident CTA slots.  Pick the
// t in 1..8 minimising  waves(t) / t * (1 + 0.1 (t - 1))  (relative time).
// Measured (profiles/r01c_tile_sweep.md): c2 t=2, c3a t=2, c3b t=3, c5 t=2,
// c4 t=1 are each the fastest of the heights swept.
int auto_tile_rows(int OH, int n_images, int slots) {
  const int n = n_images > 0 ? n_images : 1;
  int best_t = 1;
  double best = 1e30;
  for (int t = 1; t <= imin(8, ceil_div(OH, 8)); ++t) {
    const long long waves = ((long long)n * t + slots - 1) / slots;
    const double cost = (double)waves / t * (1.0 + 0.1 * (t - 1));
    if (cost < best - 1e-9) { best = cost; best_t = t; }
  }
  return ceil_div(OH, best_t);
}

int Cfg_yp(int nt) { return nt == kThreadsNarrow ? kYPNarrow : nt == kThreadsTiny ? kYPTiny : kYPWide; }

// scale 1 has no packed variant: the packed layout of scale 1 is DENSE64
KernelFn select_kernel(int K, bool f16, bool dbg, bool packed, int nt, bool db, bool gc = false,
                       bool c2s = false) {
  switch (K) {
    case 1: return select_fused_k1(f16, dbg, packed, nt, db, gc, false);
    case 2: return select_fused_k2(f16, dbg, packed, nt, db, gc, c2s);
    case 4: return select_fused_k4(f16, dbg, packed, nt, db, gc, c2s);
    default: return select_fused_k8(f16, dbg, packed, nt, db, gc, c2s);
  }
}

// Largest dynamic smem per CTA that keeps `ctas` CTAs resident per SM:
// 228 KB per SM less a 1 KB reservation per CTA, less static smem (< 512 B).
constexpr int smem_budget(int ctas) { return (228 * 1024 - ctas * 1024) / ctas - 512; }

}  // namespace

// One image's ROI block rows to gather: per component, rows [by0, by1] x
// blocks [bx0, bx1] of the (pinned host) plane -> a compact device copy.
struct GatherDesc {
  const int16_t* src[3];     // host plane (device-addressable pinned memory)
  int16_t* dst[3];           // staging
  int32_t src_stride[3];     // int16 elements per source block row
  int32_t dst_stride[3];     // int16 elements per staged row (16-B multiple)
  int32_t by0[3], rows[3];   // first ROI block row, ROI block rows
  int32_t col0[3], ncol[3];  // first ROI element in a row (bx0 * E), elements per row
};

// High-MLP copy of the ROI block rows (8-byte chunks; one CTA per image):
// PCIe reads stay in flight from every thread instead of only from the
// fused kernel's IDCT threads.
__global__ void __launch_bounds__(256) smol_gather_kernel(const GatherDesc* gd) {
  const GatherDesc g = gd[blockIdx.x];
  for (int c = 0; c < 3; ++c) {
    // 8-byte chunks covering [col0, col0 + ncol) rounded out to 4 elements;
    // source and staged rows share their alignment mod 16 B (see run_impl)
    const int a0 = g.col0[c] & ~3;
    const int nq = ((g.col0[c] + g.ncol[c] + 3) >> 2) - (a0 >> 2);
    const int total = nq * g.rows[c];
    const int16_t* src = g.src[c] + (size_t)g.by0[c] * g.src_stride[c] + a0;
    int16_t* dst = g.dst[c] - (g.col0[c] & 3);
    for (int t = threadIdx.x; t < total; t += blockDim.x) {
      const int r = t / nq, q = t - r * nq;
      const int2 v = __ldcs(reinterpret_cast<const int2*>(src + (size_t)r * g.src_stride[c]) + q);
      reinterpret_cast<int2*>(dst + (size_t)r * g.dst_stride[c])[q] = v;
    }
  }
}

struct smol_preproc_plan {
  smol_preproc_params p;
  int max_images = 0;
  int device = 0;
  int OW = 0, OH = 0;          // 0 when the output size is image dependent (never: validated)
  int tile_rows = 0;               // 0 = automatic per batch size
  int smem_optin = 0;
  int num_sms = 148;
  int min_col_tiles = 1;                  // SMOL_COL_TILES=k forces >= k column tiles (A/B)
  int nt_mode = 0;                        // SMOL_THREADS=192|256 forces the CTA size (A/B)
  DevImage* d_desc = nullptr;  // [kRing][max_images] image kinds
  DevRef* d_ref = nullptr;     // [kRing][max_images] per-image references
  int4* d_map = nullptr;       // [kRing][map_cap] balanced CTA map (see run_impl)
  int4* h_map = nullptr;       // pinned
  int map_cap = 0;
  int cta_map_mode = 1;        // SMOL_CTA_MAP=0 disables the balanced map (A/B)
  int thumb_mode = 1;          // SMOL_THUMB=0 disables the warp-per-image 1/8 kernel (A/B)
  int tap_mode = 1;            // SMOL_TAPS=0: every CTA computes its own bilinear taps (A/B)
  DevImage* h_desc = nullptr;  // pinned [kRing][max_images]
  DevRef* h_ref = nullptr;     // pinned [kRing][max_images]
  TileLayout* d_lay = nullptr; // [kRing][lay_cap] tile layouts per (kind, tile)
  TileLayout* h_lay = nullptr; // pinned
  int lay_cap = 0;
  int4* d_tap = nullptr;       // [kRing][tap_cap] bilinear tap regions per (kind, tile)
  int4* h_tap = nullptr;       // pinned
  int tap_cap = 0;             // int4 words per ring slot
  cudaEvent_t ev[kRing] = {};
  cudaEvent_t desc_ready[kRing] = {};      // descriptor upload of a ring slot done (copy stream)
  int ring = 0;
  float na[3], nb[3];
  // end-to-end (run_host / run_compact) staging: ROI block rows gathered
  // from pinned host memory (or expanded from compact records) into device
  // memory, n_stage slots deep (default 3: the host prepares run k while the
  // copy engine moves run k-1 and the SMs run k-2)
  cudaStream_t copy_stream = nullptr;
  int n_stage = kStageDefault;
  int16_t* stage[kStageMax] = {};
  size_t stage_cap[kStageMax] = {};        // bytes
  GatherDesc* d_gather = nullptr;          // [n_stage][max_images]
  GatherDesc* h_gather = nullptr;          // pinned [n_stage][max_images]
  // compact transport (run_compact): device copy of the records, expand descriptors
  uint8_t* cbuf[kStageMax] = {};
  size_t cbuf_cap[kStageMax] = {};
  ExpandDesc* d_expand = nullptr;          // [n_stage][max_images]
  ExpandDesc* h_expand = nullptr;          // pinned [n_stage][max_images]
  std::vector<TileLayout> layouts;         // host scratch (whole-output footprints)
  cudaEvent_t stage_free[kStageMax] = {}, stage_ready[kStageMax] = {};
  // run_compact: the expand kernel runs on its own stream, so batch k+1's
  // expansion fills the SMs the fused kernel of batch k leaves idle in its tail
  cudaStream_t expand_stream = nullptr;
  cudaEvent_t stage_expanded[kStageMax] = {};
  int expand_own_stream = 1;               // SMOL_EXPAND_STREAM=0: expand on `stream` (A/B)
  // run_jpeg: per staging slot the image descriptors,
  // Huffman table sets, quantization tables and the segment index
  JpegDesc* h_jdesc = nullptr;             // pinned [n_stage][max_images]
  JpegDesc* d_jdesc = nullptr;
  HuffSet* h_huff = nullptr;               // pinned [n_stage][kMaxHuffSets]
  HuffSet* d_huff = nullptr;
  uint16_t* h_jqt = nullptr;               // pinned [n_stage][kMaxJpegQt][64]
  uint16_t* d_jqt = nullptr;
  int32_t* d_seg[kStageMax] = {};          // [2][cap]: segment start byte, image
  size_t seg_cap[kStageMax] = {};          // bytes
  int8_t* d_zmap = nullptr;                // zig-zag position -> stored element of the layout (-1: dropped)
  // host scratch of the current run_jpeg call
  std::vector<JpegHdr> jhdr;               // distinct headers
  std::vector<int> jimg_hdr;               // per image: header index
  std::vector<smol_compact_image> jci;     // per image: descriptor for the common validation
  std::vector<std::array<uint16_t, 64>> jqt;   // distinct quantization tables
  std::vector<int> jhdr_set;               // per header: Huffman table set
  std::vector<std::array<int, 3>> jhdr_qid; // per header: quantization table ids per component
  std::vector<int> jset_hdr;               // per table set: a header holding it
  int jnseg = 0;                           // restart intervals of the current batch
  int jnact = 0;                           // of them holding ROI blocks (one decode thread each)
  int stage_slot = 0;
  bool fixed_stage = false;                // staging sized in plan (params.max_width/max_height)
  std::vector<std::pair<uintptr_t, uintptr_t>> pinned_ok;   // run_host: verified [lo, hi) allocations
};

extern "C" {

int32_t smol_abi_version(void) { return SMOL_ABI_VERSION; }

const char* smol_last_error(void) { return g_last_error.c_str(); }

int32_t smol_debug_geometry(const smol_preproc_params* params, const smol_image_desc* image,
                            smol_geometry* out) {
  g_last_error.clear();
  int32_t rc = validate_params(params);
  if (rc) return rc;
  if (!image || !out) return fail(SMOL_ERR_INVALID, "image/out is NULL");
  DevImage g{};
  rc = image_geometry(params, image, 0, g);
  if (rc) return rc;
  memset(out, 0, sizeof(*out));
  out->Wd = g.Wd; out->Hd = g.Hd; out->Wc = g.Wc; out->Hc = g.Hc;
  out->Wr = g.Wr; out->Hr = g.Hr; out->left = g.left; out->top = g.top;
  out->OW = params->crop_w > 0 ? params->crop_w : g.Wr;
  out->OH = params->crop_w > 0 ? params->crop_h : g.Hr;
  out->sx0 = g.sx0; out->sy0 = g.sy0; out->sw = g.sw; out->sh = g.sh;
  g.nbw[0] = ceil_div(image->width, 8);
  g.nbw[1] = g.nbw[2] = ceil_div(image->width, image->subsampling == 444 ? 8 : 16);
  TileLayout L;
  tile_layout(g, params->scale_denom, 0, out->OH, 0, out->OW, L, kYPWide, true);
  out->lx0 = L.lx0; out->lx1 = L.lx1; out->ly0 = L.ly0; out->ly1 = L.ly1;
  out->cx0 = L.cx0; out->cx1 = L.cx1; out->cy0 = L.cy0; out->cy1 = L.cy1;
  for (int c = 0; c < 3; ++c) {
    out->bx0[c] = L.bx0[c]; out->bx1[c] = L.bx1[c]; out->by0[c] = L.by0[c]; out->by1[c] = L.by1[c];
  }
  out->roi_blocks = tile_roi_blocks(L);
  // algorithmic coefficient bytes: the K_s coefficients the
  // scale uses per ROI block (reading R1: 64 / 49 / 25 / 1), 2 B each, in any
  // layout; storage bytes: what the layout holds for those blocks (PACKED
  // pads to 8 B; dense-64 at scale 1/8 reads only the DC's 32-B sector)
  out->roi_coef_bytes = 0;
  for (int c = 0; c < 3; ++c)
    out->roi_coef_bytes += (int64_t)(L.by1[c] - L.by0[c] + 1) * (L.bx1[c] - L.bx0[c] + 1) * 2 *
                           used_coefs(c ? g.ck : params->scale_denom, params->idct_def);
  const int bb = 2 * block_elems(params->scale_denom, params->layout, params->idct_def);
  out->storage_coef_bytes =
      out->roi_blocks * ((params->scale_denom == 8 && params->layout == SMOL_LAYOUT_DENSE64) ? 32 : bb);
  return SMOL_OK;
}

int32_t smol_preproc_plan(const smol_preproc_params* params, int32_t max_images, smol_preproc_plan_t** out) {
  g_last_error.clear();
  if (!out) return fail(SMOL_ERR_INVALID, "out is NULL");
  *out = nullptr;
  int32_t rc = validate_params(params);
  if (rc) return rc;
  if (max_images <= 0 || max_images > (1 << 20))
    return fail(SMOL_ERR_INVALID, "max_images=%d not in [1, 2^20]", max_images);
  int dev = 0;
  SMOL_CUDA(cudaGetDevice(&dev));
  rc = ensure_basis(dev);
  if (rc) return rc;
  {
    const long long ow = params->crop_w > 0 ? params->crop_w : params->resize_w;
    const long long oh = params->crop_w > 0 ? params->crop_h : params->resize_h;
    if (ow > 65535 || oh > 65535 || 3 * ow * oh >= (1LL << 31))
      return fail(SMOL_ERR_INVALID, "output %lldx%lld too large (3*H*W must be < 2^31 elements)", ow, oh);
  }
  smol_preproc_plan_t* pl = new (std::nothrow) smol_preproc_plan_t();
  if (!pl) return fail(SMOL_ERR_NOMEM, "plan allocation");
  pl->p = *params;
  pl->max_images = max_images;
  pl->device = dev;
  if (params->crop_w > 0) { pl->OW = params->crop_w; pl->OH = params->crop_h; }
  else { pl->OW = params->resize_w; pl->OH = params->resize_h; }
  pl->tile_rows = params->tile_rows;
  if (const char* e = std::getenv("SMOL_COL_TILES")) pl->min_col_tiles = std::atoi(e);
  if (const char* e = std::getenv("SMOL_THREADS")) pl->nt_mode = std::atoi(e);
  if (const char* e = std::getenv("SMOL_CTA_MAP")) pl->cta_map_mode = std::atoi(e);
  if (const char* e = std::getenv("SMOL_THUMB")) pl->thumb_mode = std::atoi(e);
  if (const char* e = std::getenv("SMOL_TAPS")) pl->tap_mode = std::atoi(e);
  for (int c = 0; c < 3; ++c) {
    pl->na[c] = (float)(1.0 / (255.0 * (double)params->std[c]));
    pl->nb[c] = (float)(-(double)params->mean[c] / (double)params->std[c]);
  }
  cudaError_t e = cudaDeviceGetAttribute(&pl->smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  if (e == cudaSuccess) e = cudaDeviceGetAttribute(&pl->num_sms, cudaDevAttrMultiProcessorCount, dev);
  if (e == cudaSuccess) e = cudaMalloc(&pl->d_desc, sizeof(DevImage) * (size_t)max_images * kRing);
  if (e == cudaSuccess) e = cudaMallocHost(&pl->h_desc, sizeof(DevImage) * (size_t)max_images * kRing);
  if (e == cudaSuccess) e = cudaMalloc(&pl->d_ref, sizeof(DevRef) * (size_t)max_images * kRing);
  if (e == cudaSuccess) e = cudaMallocHost(&pl->h_ref, sizeof(DevRef) * (size_t)max_images * kRing);
  pl->lay_cap = std::min(4 * max_images, 4096) + 256;
  if (e == cudaSuccess) e = cudaMalloc(&pl->d_lay, sizeof(TileLayout) * (size_t)pl->lay_cap * kRing);
  if (e == cudaSuccess) e = cudaMallocHost(&pl->h_lay, sizeof(TileLayout) * (size_t)pl->lay_cap * kRing);
  pl->tap_cap = kTapCap;
  if (e == cudaSuccess) e = cudaMalloc(&pl->d_tap, sizeof(int4) * (size_t)pl->tap_cap * kRing);
  if (e == cudaSuccess) e = cudaMallocHost(&pl->h_tap, sizeof(int4) * (size_t)pl->tap_cap * kRing);
  for (int i = 0; i < kRing && e == cudaSuccess; ++i) {
    e = cudaEventCreateWithFlags(&pl->ev[i], cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&pl->desc_ready[i], cudaEventDisableTiming);
  }
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&pl->copy_stream, cudaStreamNonBlocking);
  if (const char* ev = std::getenv("SMOL_EXPAND_STREAM")) pl->expand_own_stream = std::atoi(ev);
  if (const char* ev = std::getenv("SMOL_STAGE_SLOTS")) pl->n_stage = std::max(2, std::min(kStageMax, std::atoi(ev)));
  const size_t nst = (size_t)pl->n_stage;
  for (int i = 0; i < pl->n_stage && e == cudaSuccess; ++i) {
    e = cudaEventCreateWithFlags(&pl->stage_free[i], cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&pl->stage_ready[i], cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&pl->stage_expanded[i], cudaEventDisableTiming);
  }
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&pl->expand_stream, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaMalloc(&pl->d_gather, sizeof(GatherDesc) * (size_t)max_images * nst);
  if (e == cudaSuccess) e = cudaMallocHost(&pl->h_gather, sizeof(GatherDesc) * (size_t)max_images * nst);
  if (e == cudaSuccess) e = cudaMalloc(&pl->d_expand, sizeof(ExpandDesc) * (size_t)max_images * nst);
  if (e == cudaSuccess) e = cudaMallocHost(&pl->h_expand, sizeof(ExpandDesc) * (size_t)max_images * nst);
  if (e == cudaSuccess) e = cudaMalloc(&pl->d_jdesc, sizeof(JpegDesc) * (size_t)max_images * nst);
  if (e == cudaSuccess) e = cudaMallocHost(&pl->h_jdesc, sizeof(JpegDesc) * (size_t)max_images * nst);
  if (e == cudaSuccess) e = cudaMalloc(&pl->d_huff, sizeof(HuffSet) * kMaxHuffSets * nst);
  if (e == cudaSuccess) e = cudaMallocHost(&pl->h_huff, sizeof(HuffSet) * kMaxHuffSets * nst);
  if (e == cudaSuccess) e = cudaMalloc(&pl->d_jqt, sizeof(uint16_t) * 64 * kMaxJpegQt * nst);
  if (e == cudaSuccess) e = cudaMallocHost(&pl->h_jqt, sizeof(uint16_t) * 64 * kMaxJpegQt * nst);
  if (e == cudaSuccess) {
    // zig-zag position k (T.81 Figure A.6) -> element of the stored block:
    // dense-64: the natural index; packed: the rank of the natural index
    // among the elements the scale uses (row-major, as the PACKED layouts
    // store them), dropped (-1) if unused
    int8_t zm[64];
    const std::array<int, 64> zz = zigzag_order();
    const bool packed = params->layout == SMOL_LAYOUT_PACKED && params->scale_denom > 1;
    const uint64_t use = used_mask(params->scale_denom, false, params->idct_def == SMOL_IDCT_TRUNCATED);
    for (int k = 0; k < 64; ++k) {
      const int nat = zz[k];
      zm[k] = (int8_t)(!packed ? nat : ((use >> nat) & 1) ? __builtin_popcountll(use & ((1ull << nat) - 1)) : -1);
    }
    e = cudaMalloc(&pl->d_zmap, 64);
    if (e == cudaSuccess) e = cudaMemcpy(pl->d_zmap, zm, 64, cudaMemcpyHostToDevice);
  }
  if (e == cudaSuccess) pl->layouts.reserve(max_images);
  if (e == cudaSuccess) {
    pl->map_cap = pl->num_sms * 8;
    e = cudaMalloc(&pl->d_map, sizeof(int4) * (size_t)pl->map_cap * kRing);
    if (e == cudaSuccess) e = cudaMallocHost(&pl->h_map, sizeof(int4) * (size_t)pl->map_cap * kRing);
  }
  if (e == cudaSuccess && params->max_width > 0) {
    // staging of the staged paths for max_images images of at most
    // max_width x max_height (worst case: every block of the image, 4:4:4),
    // so run_host / run_compact never allocate: dense ROI rows (every slot)
    // and compact records (units <= 2 per used element, plus the tables)
    const int E = block_elems(params->scale_denom, params->layout, params->idct_def);
    const long long bw = ceil_div(params->max_width, 8), bh = ceil_div(params->max_height, 8);
    const long long rows = 3 * bh, blocks = 3 * bw * bh;
    const size_t stage_img = (size_t)(2 * (blocks * E + rows * 16 + 3 * 8));
    const size_t rec_img = (size_t)compact_record_bytes(blocks, rows, 2LL * blocks * used_coefs(params->scale_denom, params->idct_def));
    for (int i = 0; i < pl->n_stage && e == cudaSuccess; ++i) {
      pl->stage_cap[i] = stage_img * (size_t)max_images;
      e = cudaMalloc(&pl->stage[i], pl->stage_cap[i] + 256);
      if (e == cudaSuccess) {
        pl->cbuf_cap[i] = rec_img * (size_t)max_images;
        e = cudaMalloc(&pl->cbuf[i], pl->cbuf_cap[i] + 256);
      }
    }
    // run_jpeg segment index: at most one restart interval per MCU (8x8 px
    // worst case), 3 int32 each (start, image, active list) + the counter
    const size_t seg_img = (size_t)12 * ceil_div(params->max_width, 8) * ceil_div(params->max_height, 8);
    for (int i = 0; i < pl->n_stage && e == cudaSuccess; ++i) {
      pl->seg_cap[i] = seg_img * (size_t)max_images + 16;
      e = cudaMalloc(&pl->d_seg[i], pl->seg_cap[i] + 256);
    }
    pl->fixed_stage = true;
  }
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(smol_expand_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kExpandSmem);
  if (e == cudaSuccess) {
    // opt every instantiation of this plan's (scale, dtype) in to the largest
    // dynamic smem the device allows next to the kernel's static smem
    const bool f16 = params->out_dtype == SMOL_OUT_F16_NCHW;
    int limit = pl->smem_optin;
    for (int v = 0; v < 10 && e == cudaSuccess; ++v) {
      if (v >= 8 && !params->chroma_2s) break;
      const int dbg = v & 1, nt = v < 2 ? kThreadsWide : v < 4 ? kThreadsNarrow : kThreadsTiny;
      cudaFuncAttributes fa;
      KernelFn fn = select_kernel(params->scale_denom, f16, dbg, params->layout == SMOL_LAYOUT_PACKED, nt,
                                  params->idct_def == SMOL_IDCT_TRUNCATED, v >= 6, v >= 8);
      e = cudaFuncGetAttributes(&fa, fn);
      if (e != cudaSuccess) break;
      const int dyn = pl->smem_optin - (int)fa.sharedSizeBytes;
      if (dyn < limit) limit = dyn;
      e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, dyn);
    }
    pl->smem_optin = limit;
  }
  if (e != cudaSuccess) {
    smol_preproc_destroy(pl);
    return fail(e == cudaErrorMemoryAllocation ? SMOL_ERR_NOMEM : SMOL_ERR_CUDA, "plan setup: %s",
                cudaGetErrorString(e));
  }
  *out = pl;
  return SMOL_OK;
}

void smol_preproc_destroy(smol_preproc_plan_t* pl) {
  if (!pl) return;
  int prev = -1;                    // release on the plan's device, then restore the caller's
  if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
  if (prev != pl->device) cudaSetDevice(pl->device);
  for (int i = 0; i < kRing; ++i) {
    if (pl->ev[i]) { cudaEventSynchronize(pl->ev[i]); cudaEventDestroy(pl->ev[i]); }
    if (pl->desc_ready[i]) cudaEventDestroy(pl->desc_ready[i]);
  }
  for (int i = 0; i < kStageMax; ++i) {
    if (pl->stage_free[i]) { cudaEventSynchronize(pl->stage_free[i]); cudaEventDestroy(pl->stage_free[i]); }
    if (pl->stage_ready[i]) cudaEventDestroy(pl->stage_ready[i]);
    if (pl->stage_expanded[i]) cudaEventDestroy(pl->stage_expanded[i]);
    if (pl->stage[i]) cudaFree(pl->stage[i]);
    if (pl->cbuf[i]) cudaFree(pl->cbuf[i]);
  }
  for (int i = 0; i < kStageMax; ++i)
    if (pl->d_seg[i]) cudaFree(pl->d_seg[i]);
  if (pl->d_jdesc) cudaFree(pl->d_jdesc);
  if (pl->h_jdesc) cudaFreeHost(pl->h_jdesc);
  if (pl->d_huff) cudaFree(pl->d_huff);
  if (pl->h_huff) cudaFreeHost(pl->h_huff);
  if (pl->d_jqt) cudaFree(pl->d_jqt);
  if (pl->h_jqt) cudaFreeHost(pl->h_jqt);
  if (pl->d_zmap) cudaFree(pl->d_zmap);
  if (pl->d_expand) cudaFree(pl->d_expand);
  if (pl->h_expand) cudaFreeHost(pl->h_expand);
  if (pl->d_gather) cudaFree(pl->d_gather);
  if (pl->h_gather) cudaFreeHost(pl->h_gather);
  if (pl->copy_stream) cudaStreamDestroy(pl->copy_stream);
  if (pl->expand_stream) cudaStreamDestroy(pl->expand_stream);
  if (pl->d_desc) cudaFree(pl->d_desc);
  if (pl->d_map) cudaFree(pl->d_map);
  if (pl->h_map) cudaFreeHost(pl->h_map);
  if (pl->h_desc) cudaFreeHost(pl->h_desc);
  if (pl->d_ref) cudaFree(pl->d_ref);
  if (pl->d_lay) cudaFree(pl->d_lay);
  if (pl->h_lay) cudaFreeHost(pl->h_lay);
  if (pl->d_tap) cudaFree(pl->d_tap);
  if (pl->h_tap) cudaFreeHost(pl->h_tap);
  if (pl->h_ref) cudaFreeHost(pl->h_ref);
  const int dev = pl->device;
  delete pl;
  if (prev >= 0 && prev != dev) cudaSetDevice(prev);
}

int32_t smol_preproc_output_shape(const smol_preproc_plan_t* pl, int32_t* c, int32_t* h, int32_t* w) {
  if (!pl || !c || !h || !w) return fail(SMOL_ERR_INVALID, "NULL argument");
  *c = 3; *h = pl->OH; *w = pl->OW;
  return SMOL_OK;
}

int32_t smol_preproc_launches_per_run(const smol_preproc_plan_t* pl) {
  return pl ? 1 : 0;
}

}  // extern "C"

namespace {

// Where the coefficient blocks come from.
enum class Src { kDevice, kGather, kCompact, kJpeg };

// Validate a compact image descriptor into its device descriptor (coefficient
// pointers are set by the staging step).
int32_t validate_compact_image(const smol_preproc_params* p, const smol_compact_image* ci, int idx,
                               int n_qtables, DevImage& g, const DevImage* geom = nullptr) {
  if (geom) {
    copy_geometry(*geom, g);
  } else {
    smol_image_desc d{};
    d.width = ci->width; d.height = ci->height; d.subsampling = ci->subsampling;
    d.roi_left = ci->roi_left; d.roi_top = ci->roi_top;
    d.roi_x = ci->roi_x; d.roi_y = ci->roi_y; d.roi_w = ci->roi_w; d.roi_h = ci->roi_h;
    int32_t rc = image_geometry(p, &d, idx, g);
    if (rc) return rc;
  }
  if (ci->offset < 0 || ci->offset % 16)
    return fail(SMOL_ERR_INVALID, "image %d: record offset %lld not a non-negative multiple of 16", idx,
                (long long)ci->offset);
  for (int c = 0; c < 3; ++c) {
    g.qidx[c] = 0;
    if (!(c > 0 && g.gray)) {
      if (ci->qtable[c] < 0 || ci->qtable[c] >= n_qtables)
        return fail(SMOL_ERR_INVALID, "image %d: qtable[%d]=%d not in [0,%d)", idx, c, ci->qtable[c], n_qtables);
      g.qidx[c] = ci->qtable[c];
    }
    g.nbw[c] = ceil_div(ci->width, c ? (ci->subsampling == 444 ? 8 : 16) : 8);
    g.coef[c] = nullptr;
    g.stride[c] = 0;
  }
  return SMOL_OK;
}

// Staged-plane layout of one image's ROI block rows (whole-output footprint):
// per component rows [by0, by1] x elements [bx0 E, (bx1 + 1) E), each row
// padded to 16 B with a leading pad so the kernel's virtual row base
// (row - col0) is 16-B aligned, as for an original plane (its L2 bulk
// prefetch needs it).  Returns the staged int16 elements; offsets in dst_off.
size_t stage_layout(const TileLayout& L, int E, int32_t (&dst_stride)[3], size_t (&dst_off)[3], size_t need) {
  for (int c = 0; c < 3; ++c) {
    const int ncol = (L.bx1[c] - L.bx0[c] + 1) * E;
    const int pad = (L.bx0[c] * E) & 7;
    dst_stride[c] = (pad + ncol + 7) & ~7;
    dst_off[c] = need + pad;
    need += (size_t)dst_stride[c] * (L.by1[c] - L.by0[c] + 1);
  }
  return need;
}

int32_t grow(void** buf, size_t* cap, size_t need, cudaStream_t s, bool fixed, const char* what) {
  if (need <= *cap) return SMOL_OK;
  if (fixed)                       // sized in plan from params.max_width/max_height: never allocate here
    return fail(SMOL_ERR_CAPACITY, "%s needs %zu B > %zu B sized in plan (params.max_width/max_height)",
                what, need, *cap);
  SMOL_CUDA(cudaStreamSynchronize(s));
  if (*buf) SMOL_CUDA(cudaFree(*buf));
  *buf = nullptr;
  *cap = 0;
  SMOL_CUDA(cudaMalloc(buf, need + 256));
  *cap = need;
  return SMOL_OK;
}

int32_t run_impl(smol_preproc_plan_t* pl, int n_images, const void* images, const uint16_t* qtables,
                 int n_qtables, void* out, void* stream_v, const KParams* dbg, Src src,
                 const smol_compact_batch* cb = nullptr, const smol_jpeg_batch* jb = nullptr) {
  // (run_jpeg calls with its parsed descriptors and no g_last_error reset:
  // its own messages so far are kept only on failure)
  if (src != Src::kJpeg) g_last_error.clear();
  if (n_images < 0) return fail(SMOL_ERR_INVALID, "n_images=%d < 0", n_images);
  if (n_images == 0) return SMOL_OK;
  if (n_images > pl->max_images)
    return fail(SMOL_ERR_CAPACITY, "n_images=%d > plan capacity %d", n_images, pl->max_images);
  if (!images) return fail(SMOL_ERR_INVALID, "batch.images is NULL");
  if ((!qtables && src != Src::kJpeg) || n_qtables < 1 || n_qtables > (src == Src::kJpeg ? kMaxJpegQt : 4))
    return fail(SMOL_ERR_INVALID, "batch.qtables NULL or n_qtables=%d not in [1,4]", n_qtables);
  if (!out) return fail(SMOL_ERR_INVALID, "out is NULL");
  {
    int cur = -1;
    SMOL_CUDA(cudaGetDevice(&cur));
    if (cur != pl->device)
      return fail(SMOL_ERR_INVALID, "plan was created on device %d but device %d is current", pl->device, cur);
  }
  const size_t out_esz = pl->p.out_dtype == SMOL_OUT_F16_NCHW ? 2 : 4;
  if (reinterpret_cast<uintptr_t>(out) % out_esz)
    return fail(SMOL_ERR_INVALID, "out is not %zu-byte aligned", out_esz);
  cudaStream_t stream = reinterpret_cast<cudaStream_t>(stream_v);
  const int K = pl->p.scale_denom;
  const bool packed = pl->p.layout == SMOL_LAYOUT_PACKED;

  // ring slot: wait until the run that last used it has consumed its descriptors
  const int slot = pl->ring;
  pl->ring = (pl->ring + 1) % kRing;
  SMOL_CUDA(cudaEventSynchronize(pl->ev[slot]));
  DevImage* h = pl->h_desc + (size_t)slot * pl->max_images;   // kinds
  DevImage* d = pl->d_desc + (size_t)slot * pl->max_images;
  DevRef* hr = pl->h_ref + (size_t)slot * pl->max_images;      // per image
  DevRef* dr = pl->d_ref + (size_t)slot * pl->max_images;

  // provisional tile height (4 CTAs per SM); final once the CTA size is known
  const bool auto_rows = pl->tile_rows <= 0;
  int tile_rows = auto_rows ? auto_tile_rows(pl->OH, n_images, pl->num_sms * 4) : imin(pl->tile_rows, pl->OH);
  int ntiles = ceil_div(pl->OH, tile_rows);
  // validate every descriptor once; consecutive images whose descriptors
  // differ only in their coefficient pointers (compact: record offsets)
  // share one kind, so per image only the pointers are checked and written
  int nk = 0;
  for (int i = 0; i < n_images; ++i) {
    int32_t rc = SMOL_OK;
    if (src == Src::kCompact || src == Src::kJpeg) {
      const smol_compact_image* ci = static_cast<const smol_compact_image*>(images);
      const bool same = i > 0 && memcmp(&ci[i], &ci[i - 1], offsetof(smol_compact_image, offset)) == 0;
      if (!same) {
        const bool sg = i > 0 && ci[i].width == ci[i - 1].width && ci[i].height == ci[i - 1].height &&
                        ci[i].subsampling == ci[i - 1].subsampling && ci[i].roi_left == ci[i - 1].roi_left &&
                        ci[i].roi_top == ci[i - 1].roi_top && ci[i].roi_x == ci[i - 1].roi_x &&
                        ci[i].roi_y == ci[i - 1].roi_y && ci[i].roi_w == ci[i - 1].roi_w &&
                        ci[i].roi_h == ci[i - 1].roi_h;
        rc = validate_compact_image(&pl->p, &ci[i], i, n_qtables, h[nk], sg ? &h[nk - 1] : nullptr);
        ++nk;
      } else if (ci[i].offset < 0 || ci[i].offset % 16) {
        rc = fail(SMOL_ERR_INVALID, "image %d: record offset %lld not a non-negative multiple of 16", i,
                  (long long)ci[i].offset);
      }
      hr[i].kind = nk - 1;
      hr[i].coef[0] = hr[i].coef[1] = hr[i].coef[2] = nullptr;
    } else {
      const smol_image_desc* di = static_cast<const smol_image_desc*>(images);
      // (fields before and after the coefficient pointers)
      const bool same = i > 0 && memcmp(&di[i], &di[i - 1], offsetof(smol_image_desc, coef)) == 0 &&
                        memcmp(&di[i].blocks_w, &di[i - 1].blocks_w,
                               sizeof(smol_image_desc) - offsetof(smol_image_desc, blocks_w)) == 0;
      if (!same) {
        const bool sg = i > 0 && same_geometry(&di[i], &di[i - 1]);
        rc = validate_image(&pl->p, &di[i], i, n_qtables, h[nk], true, sg ? &h[nk - 1] : nullptr);
        ++nk;
      } else {
        for (int c = 0; c < (h[nk - 1].gray ? 1 : 3) && !rc; ++c)
          if (!di[i].coef[c] || reinterpret_cast<uintptr_t>(di[i].coef[c]) % 16)
            rc = fail(SMOL_ERR_INVALID, "image %d: coef[%d] NULL or not 16-byte aligned", i, c);
      }
      hr[i].kind = nk - 1;
      const bool gray = h[nk - 1].gray;
      hr[i].coef[0] = di[i].coef[0];
      hr[i].coef[1] = gray ? nullptr : di[i].coef[1];
      hr[i].coef[2] = gray ? nullptr : di[i].coef[2];
    }
    if (rc) return rc;
  }
  // shared memory of the largest tile over the batch's distinct geometries
  // (a tile whose footprint exceeds the fixed ring pitches reports INT_MAX/2)
  auto cols_of = [&](int n_col_tiles) { return (ceil_div(pl->OW, n_col_tiles) + 3) & ~3; };  // multiple of 4
  // a batch with any 4:2:2 / 4:4:4 image runs the generic-chroma kernel
  // (wide CTA only; its chroma rings are full-size)
  bool gc = false;
  for (int i = 0; i < nk && !gc; ++i) gc = h[i].hs != 2 || h[i].vs != 2;
  auto max_smem = [&](int n_col_tiles, int yp) {
    const int tile_cols = cols_of(n_col_tiles);
    n_col_tiles = ceil_div(pl->OW, tile_cols);
    int m = 0;
    const DevImage* prev = nullptr;
    for (int i = 0; i < nk; ++i) {
      const DevImage& g = h[i];
      if (prev && same_layout_inputs(g, *prev)) continue;
      for (int t = 0; t < ntiles; ++t)
        for (int u = 0; u < n_col_tiles; ++u) {
          TileLayout L;
          tile_layout(g, K, t * tile_rows, imin(pl->OH, (t + 1) * tile_rows), u * tile_cols,
                      imin(pl->OW, (u + 1) * tile_cols), L, yp, gc);
          m = imax(m, L.fits ? L.total : (1 << 30));
        }
      prev = &g;
    }
    return m;
  };
  // Tiny configuration (128 threads, 128-B rings, 6 CTAs/SM) for small
  // footprints, narrow (192 threads, 384-B ring pitch) when full-width tiles
  // fit it with 4 CTAs per SM; otherwise wide (256 threads, 512-B pitch),
  // adding column tiles only when a tile would not leave 2 CTAs/SM.
  int n_col_tiles = 1;
  int nt = kThreadsTiny;
  int smem = gc ? INT_MAX : max_smem(1, kYPTiny);
  if (smem > smem_budget(6) || (pl->nt_mode != 0 && pl->nt_mode != kThreadsTiny) || pl->min_col_tiles > 1) {
    nt = kThreadsNarrow;
    smem = gc ? INT_MAX : max_smem(1, kYPNarrow);
  }
  if (smem > smem_budget(4) || pl->nt_mode == kThreadsWide || pl->min_col_tiles > 1) {
    nt = kThreadsWide;
    smem = max_smem(1, kYPWide);
    while (smem > pl->smem_optin / 2 && n_col_tiles < 64 && 8 * n_col_tiles <= pl->OW) {
      n_col_tiles *= 2;
      smem = max_smem(n_col_tiles, kYPWide);
    }
    if (pl->min_col_tiles > n_col_tiles && 8 * pl->min_col_tiles <= pl->OW) {   // A/B override
      n_col_tiles = pl->min_col_tiles;
      smem = max_smem(n_col_tiles, kYPWide);
    }
  }
  // resident CTAs per SM of the chosen kernel at this shared-memory size
  bool c2s = false;                        // some image decodes chroma at twice the scale (R18)
  for (int i = 0; i < nk && !c2s; ++i) c2s = h[i].ck != K;
  KernelFn fn = select_kernel(K, pl->p.out_dtype == SMOL_OUT_F16_NCHW, dbg != nullptr, packed, nt,
                              pl->p.idct_def == SMOL_IDCT_TRUNCATED, gc, c2s);
  const int cta_threads = nt;
  int occ = 768 / cta_threads;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, cta_threads, smem) != cudaSuccess || occ < 1) {
    cudaGetLastError();
    occ = 768 / cta_threads;
  }
  if (auto_rows && n_col_tiles == 1) {
    const int tr = auto_tile_rows(pl->OH, n_images, pl->num_sms * occ);
    if (tr != tile_rows) {
      tile_rows = tr;
      ntiles = ceil_div(pl->OH, tile_rows);
      smem = max_smem(1, Cfg_yp(nt));
    }
  }
  {
    // the kernel's magic-number divisions (FastDiv) are exact for n * d <
    // 2^32: output task indices reach tile_rows * nq4 with divisor nq4
    const long long nq4 = (cols_of(n_col_tiles) + 3) / 4;
    const long long cap = 0xFFFFFFFFLL / (nq4 * nq4);
    if (tile_rows > cap) {
      tile_rows = (int)std::max<long long>(1, cap);
      ntiles = ceil_div(pl->OH, tile_rows);
    }
  }
  // Scale 1/8 with small footprints (thumbnails): the warp-per-image kernel
  // (smol_thumb.cuh) when every distinct geometry fits its per-warp buffers.
  // Packed layout only: with dense-64 blocks each DC is a separate 32-B
  // sector and the tiled kernel hides that latency better (measured r01s:
  // c4 packed 47.5 M -> 52.1 M img/s, dense 33.6 M -> 27.0 M).
  bool thumb = K == 8 && packed && !dbg && !gc && pl->thumb_mode && pl->OW <= kThumbMaxOut &&
               pl->OH <= kThumbMaxOut;
  for (int i = 0; thumb && i < nk; ++i) {
    if (i > 0 && same_layout_inputs(h[i], h[i - 1])) continue;
    TileLayout L;
    tile_layout(h[i], K, 0, pl->OH, 0, pl->OW, L, kYPTiny);
    thumb = L.lx1 - L.lx0 + 1 <= kThumbMaxFoot && L.ly1 - L.ly0 + 1 <= kThumbMaxFoot &&
            L.cx1 - L.cx0 + 1 <= kThumbCP && L.cy1 - L.cy0 + 1 <= kThumbCP;
  }
  // Balanced CTA map: when the automatic tiling leaves one partial wave
  // (n * t CTAs < resident slots S), give S - n t images one more (shorter)
  // tile so every slot is busy, and launch the taller tiles first.  The time
  // is set by the SMs holding the most work; with 512 tiles of 112 rows on
  // 592 slots (c2) those hold 4 tiles while others hold 3.
  int map_n = 0;
  int4* hm = pl->h_map + (size_t)slot * pl->map_cap;
  int4* dm = pl->d_map + (size_t)slot * pl->map_cap;
  // (all scales: r02n c3a 0.0698 -> 0.0672 ms, c3b 0.0374 -> 0.0369, c5
  // unchanged; round 1 had measured the halos costing more at 1/2..1/8,
  // r01m, before the per-kind tile layouts and tap tables)
  if (pl->cta_map_mode && auto_rows && n_col_tiles == 1 && !thumb) {
    const int S = pl->num_sms * occ;
    const long long base = (long long)n_images * ntiles;
    if (base < S && S <= pl->map_cap && ntiles + 1 <= pl->OH / 8) {
      const int extra = (int)std::min<long long>(S - base, n_images);   // images with ntiles + 1 tiles
      for (int pass = 0; pass < 2; ++pass)          // taller tiles (ntiles per image) first
        for (int i = pass == 0 ? extra : 0; i < (pass == 0 ? n_images : extra); ++i) {
          const int t = ntiles + (i < extra ? 1 : 0);
          for (int j = 0; j < t; ++j)
            hm[map_n++] = make_int4(i, (int)((long long)j * pl->OH / t), (int)((long long)(j + 1) * pl->OH / t),
                                    t == ntiles ? j : ntiles + j);      // layout: t-tile slot j
        }
      smem += 64;      // tile positions differ from the uniform grid's: one step of slack
    }
  }
  if (smem > pl->smem_optin)
    return fail(SMOL_ERR_CAPACITY, "tile needs %d B of shared memory > %d; lower tile_rows", smem, pl->smem_optin);

  // Tile layouts per (image kind, tile), so no CTA (or thumbnail warp)
  // computes its own with a serial lane: the grid's row x column tiles, the
  // balanced map's t- and (t+1)-tile splits, or the thumbnail's one tile.
  // (Left to the kernel when the table would not fit its ring slot.)
  const int lay_stride = thumb ? 1 : map_n ? 2 * ntiles + 1 : ntiles * n_col_tiles;
  TileLayout* hl = pl->h_lay + (size_t)slot * pl->lay_cap;
  TileLayout* dl = pl->d_lay + (size_t)slot * pl->lay_cap;
  int nl = (long long)nk * lay_stride <= pl->lay_cap ? nk * lay_stride : 0;
  {
    const int tcols = cols_of(n_col_tiles), yp = thumb ? kYPTiny : Cfg_yp(nt);
    for (int k = 0; k < nk && nl; ++k)
      for (int j = 0; j < lay_stride; ++j) {
        int oy0 = 0, oy1 = pl->OH, ox0 = 0, ox1 = pl->OW;
        if (map_n) {                         // slot j < ntiles: j of ntiles; else j - ntiles of ntiles + 1
          const int t = j < ntiles ? ntiles : ntiles + 1, jj = j < ntiles ? j : j - ntiles;
          oy0 = (int)((long long)jj * pl->OH / t); oy1 = (int)((long long)(jj + 1) * pl->OH / t);
        } else if (!thumb) {
          const int trow = j / n_col_tiles, tcol = j - trow * n_col_tiles;
          oy0 = trow * tile_rows; oy1 = imin(pl->OH, oy0 + tile_rows);
          ox0 = tcol * tcols; ox1 = imin(pl->OW, ox0 + tcols);
        }
        tile_layout(h[k], K, oy0, oy1, ox0, ox1, hl[(size_t)k * lay_stride + j], yp, gc && !thumb);
      }
  }
  // Bilinear taps per (image kind, tile), in the layout of the tile's
  // shared-memory tap region, so a CTA copies them in instead of dividing
  // per output row and column (the same smol_geom.cuh functions either way:
  // same bits).  Bounded by kTapCap; tiles past it compute their own.
  int ntap = 0;
  int4* ht = pl->h_tap + (size_t)slot * pl->tap_cap;
  int4* dt = pl->d_tap + (size_t)slot * pl->tap_cap;
  if (pl->tap_mode) {
    const int pitch4 = rgb_pitch(thumb ? kYPTiny : Cfg_yp(nt)) * 4;
    for (int j = 0; j < nl; ++j) {
      TileLayout& L = hl[j];
      const DevImage& im = h[j / lay_stride];
      const int words = thumb ? thumb_tap_words(pl->OW, pl->OH) : tile_tap_bytes(L) / 16;
      if (ntap + words > pl->tap_cap) break;
      int* e = reinterpret_cast<int*>(ht + ntap);
      memset(e, 0, sizeof(int4) * (size_t)words);
      if (thumb) {
        const int nxp = (pl->OW + 1) >> 1;
        for (int q = 0; q < nxp; ++q) thumb_xp(im, L, pl->OW, q, e + 4 * q);
        for (int i = 0; i < pl->OH; ++i) thumb_yt(im, L, i, e + 4 * nxp + 2 * i);
      } else {
        const int nq4 = (L.ox1 - L.ox0 + 3) >> 2;
        for (int i = 0; i < 4 * nq4; ++i) tile_xtap(im, L, i, e);
        int* yt = e + (L.off_yt - L.off_xt) / 4;
        for (int i = 0; i < L.oy1 - L.oy0; ++i) tile_ytap(im, L, i, pitch4, yt);
      }
      L.tap_off = ntap;
      ntap += words;
    }
  }

  int sl_used = -1;                 // staging slot of a staged run
  if (src != Src::kDevice) {
    // Staged paths: each image's ROI block rows (the whole output's tap
    // footprint) are rebuilt in a plan-owned device buffer on the plan's copy
    // stream -- gathered from pinned host planes (kGather) or expanded from
    // compact records (kCompact) -- then the descriptors point at it.
    const int sl = pl->stage_slot;
    sl_used = sl;
    pl->stage_slot = (sl + 1) % pl->n_stage;
    SMOL_CUDA(cudaEventSynchronize(pl->stage_free[sl]));     // host side: descriptor slot reusable
    const int E = block_elems(K, pl->p.layout, pl->p.idct_def);
    GatherDesc* hg = pl->h_gather + (size_t)sl * pl->max_images;
    GatherDesc* dg = pl->d_gather + (size_t)sl * pl->max_images;
    ExpandDesc* he = pl->h_expand + (size_t)sl * pl->max_images;
    ExpandDesc* de = pl->d_expand + (size_t)sl * pl->max_images;
    size_t need = 0;
    size_t offs[3];
    int32_t strides[3];
    std::vector<TileLayout>& Ls = pl->layouts;      // per kind (images of a kind share their ROI ranges)
    Ls.resize(nk);
    for (int k = 0; k < nk; ++k) {
      if (k > 0 && same_layout_inputs(h[k], h[k - 1])) Ls[k] = Ls[k - 1];
      else tile_layout(h[k], K, 0, pl->OH, 0, pl->OW, Ls[k], kYPWide, true);
    }
    for (int i = 0; i < n_images; ++i) {
      const int kd = hr[i].kind;
      const TileLayout& L = Ls[kd];
      need = stage_layout(L, E, strides, offs, need);
      for (int c = 0; c < 3; ++c) {
        if (src == Src::kGather) {
          GatherDesc& g = hg[i];
          const smol_image_desc& di = static_cast<const smol_image_desc*>(images)[i];
          g.src[c] = hr[i].coef[c];
          g.src_stride[c] = di.row_stride_bytes[c] / 2;
          g.by0[c] = L.by0[c];
          g.rows[c] = L.by1[c] - L.by0[c] + 1;
          g.col0[c] = L.bx0[c] * E;
          g.ncol[c] = (L.bx1[c] - L.bx0[c] + 1) * E;
          g.dst_stride[c] = strides[c];
          g.dst[c] = reinterpret_cast<int16_t*>(offs[c]);          // offset; rebased below
        } else {
          ExpandDesc& e = he[i];
          e.dst[c] = reinterpret_cast<int16_t*>(offs[c]);
          e.dst_stride[c] = strides[c];
          e.nbx[c] = L.bx1[c] - L.bx0[c] + 1;
          e.nby[c] = L.by1[c] - L.by0[c] + 1;
          e.E = E;
        }
      }
    }
    for (int k = 0; k < nk; ++k)            // staged planes: the kind's rows have the staged stride
      stage_layout(Ls[k], E, h[k].stride, offs, 0);
    void* sbuf = pl->stage[sl];
    int32_t rc = grow(&sbuf, &pl->stage_cap[sl], need * 2, pl->copy_stream, pl->fixed_stage, "staging");
    pl->stage[sl] = static_cast<int16_t*>(sbuf);
    if (rc) return rc;
    int16_t* base = pl->stage[sl];
    for (int i = 0; i < n_images; ++i) {
      const int kd = hr[i].kind;
      const TileLayout& L = Ls[kd];
      for (int c = 0; c < 3; ++c) {
        int16_t** dp = src == Src::kGather ? &hg[i].dst[c] : &he[i].dst[c];
        *dp = base + reinterpret_cast<size_t>(*dp);
        // reference to the staged plane: same absolute block indexing
        hr[i].coef[c] = *dp - (ptrdiff_t)L.by0[c] * h[kd].stride[c] - (ptrdiff_t)L.bx0[c] * E;
      }
    }
    // Every host->device copy of a staged run goes on the copy stream, small
    // descriptors first: an H2D copy on `stream` would queue in the copy
    // engine behind the next batch's bulk transfer and serialise the pipeline.
    SMOL_CUDA(cudaStreamWaitEvent(pl->copy_stream, pl->stage_free[sl], 0));   // previous user done
    if (src == Src::kGather) {
      SMOL_CUDA(cudaMemcpyAsync(dg, hg, sizeof(GatherDesc) * n_images, cudaMemcpyHostToDevice, pl->copy_stream));
      SMOL_CUDA(cudaMemcpyAsync(d, h, sizeof(DevImage) * nk, cudaMemcpyHostToDevice, pl->copy_stream));
      SMOL_CUDA(cudaMemcpyAsync(dr, hr, sizeof(DevRef) * n_images, cudaMemcpyHostToDevice, pl->copy_stream));
      if (nl) SMOL_CUDA(cudaMemcpyAsync(dl, hl, sizeof(TileLayout) * nl, cudaMemcpyHostToDevice, pl->copy_stream));
      if (ntap) SMOL_CUDA(cudaMemcpyAsync(dt, ht, sizeof(int4) * ntap, cudaMemcpyHostToDevice, pl->copy_stream));
      smol_gather_kernel<<<n_images, 256, 0, pl->copy_stream>>>(dg);
      SMOL_CUDA(cudaGetLastError());
    } else if (src == Src::kCompact) {
      // records: bounds (and, for host arenas, header) checks, then one DMA of
      // the batch's byte range
      const smol_compact_image* ci = static_cast<const smol_compact_image*>(images);
      cudaPointerAttributes pa;
      if (cudaPointerGetAttributes(&pa, cb->arena) != cudaSuccess) {
        cudaGetLastError();
        return fail(SMOL_ERR_INVALID, "compact arena is neither host nor device memory");
      }
      const bool on_device = pa.type == cudaMemoryTypeDevice || pa.type == cudaMemoryTypeManaged;
      const uint8_t* arena = static_cast<const uint8_t*>(cb->arena);
      int64_t lo = INT64_MAX, hi = 0;
      for (int i = 0; i < n_images; ++i) {
        const ExpandDesc& e = he[i];
        int64_t nblocks = 0, nrows = 0;
        for (int c = 0; c < 3; ++c) { nblocks += (int64_t)e.nbx[c] * e.nby[c]; nrows += e.nby[c]; }
        int64_t bytes = compact_entries_off(nblocks, nrows);
        if (ci[i].offset + bytes > cb->arena_bytes)
          return fail(SMOL_ERR_INVALID, "image %d: record at %lld (>= %lld B) outside arena of %lld B", i,
                      (long long)ci[i].offset, (long long)bytes, (long long)cb->arena_bytes);
        if (!on_device) {
          CompactHeader hd;
          memcpy(&hd, arena + ci[i].offset, sizeof(hd));
          bool ok = hd.magic == kCompactMagic && (int)hd.E == E;
          for (int c = 0; c < 3 && ok; ++c)
            ok = hd.bx0[c] == Ls[hr[i].kind].bx0[c] && hd.by0[c] == Ls[hr[i].kind].by0[c] && hd.nbx[c] == e.nbx[c] &&
                 hd.nby[c] == e.nby[c];
          if (!ok)
            return fail(SMOL_ERR_INVALID, "image %d: compact record header does not match this plan's "
                        "layout/ROI (bad magic, E or block ranges)", i);
          bytes = compact_record_bytes(nblocks, nrows, hd.n_units);
          if (ci[i].offset + bytes > cb->arena_bytes)
            return fail(SMOL_ERR_INVALID, "image %d: record (%lld B) overruns the arena", i, (long long)bytes);
          // (block lengths and row starts are clamped inside the expand
          // kernel: a corrupt record yields wrong samples, never an
          // out-of-bounds access -- no per-byte host pass on the e2e path)
        }
        lo = std::min<int64_t>(lo, ci[i].offset);
        hi = std::max<int64_t>(hi, ci[i].offset + bytes);
      }
      const uint8_t* rec_base = arena;
      if (on_device) {
        lo = 0;
      } else {
        void* cbuf = pl->cbuf[sl];
        rc = grow(&cbuf, &pl->cbuf_cap[sl], (size_t)(hi - lo), pl->copy_stream, pl->fixed_stage,
                  "compact records");
        pl->cbuf[sl] = static_cast<uint8_t*>(cbuf);
        if (rc) return rc;
        rec_base = pl->cbuf[sl];
      }
      for (int i = 0; i < n_images; ++i) he[i].rec = rec_base + (ci[i].offset - lo);
      SMOL_CUDA(cudaMemcpyAsync(de, he, sizeof(ExpandDesc) * n_images, cudaMemcpyHostToDevice, pl->copy_stream));
      SMOL_CUDA(cudaMemcpyAsync(d, h, sizeof(DevImage) * nk, cudaMemcpyHostToDevice, pl->copy_stream));
      SMOL_CUDA(cudaMemcpyAsync(dr, hr, sizeof(DevRef) * n_images, cudaMemcpyHostToDevice, pl->copy_stream));
      if (nl) SMOL_CUDA(cudaMemcpyAsync(dl, hl, sizeof(TileLayout) * nl, cudaMemcpyHostToDevice, pl->copy_stream));
      if (ntap) SMOL_CUDA(cudaMemcpyAsync(dt, ht, sizeof(int4) * ntap, cudaMemcpyHostToDevice, pl->copy_stream));
      if (!on_device)
        SMOL_CUDA(cudaMemcpyAsync(pl->cbuf[sl], arena + lo, (size_t)(hi - lo), cudaMemcpyHostToDevice,
                                  pl->copy_stream));
    } else {
      // JPEG files (N4): per image the decoder descriptor (staged ROI box
      // from the expand descriptor, header fields, table set), the distinct
      // quantization tables and Huffman table sets, then one DMA of the
      // batch's byte range
      const smol_jpeg_image* ji = jb->images;
      const uint8_t* arena = static_cast<const uint8_t*>(jb->arena);
      int64_t lo = INT64_MAX, hi = 0;
      for (int i = 0; i < n_images; ++i) {
        lo = std::min<int64_t>(lo, ji[i].offset);
        hi = std::max<int64_t>(hi, ji[i].offset + ji[i].size);
      }
      void* cbuf = pl->cbuf[sl];
      rc = grow(&cbuf, &pl->cbuf_cap[sl], (size_t)(hi - lo), pl->copy_stream, pl->fixed_stage, "JPEG files");
      pl->cbuf[sl] = static_cast<uint8_t*>(cbuf);
      if (rc) return rc;
      JpegDesc* hj = pl->h_jdesc + (size_t)sl * pl->max_images;
      JpegDesc* dj = pl->d_jdesc + (size_t)sl * pl->max_images;
      HuffSet* hh = pl->h_huff + (size_t)sl * kMaxHuffSets;
      HuffSet* dh = pl->d_huff + (size_t)sl * kMaxHuffSets;
      uint16_t* hq = pl->h_jqt + (size_t)sl * kMaxJpegQt * 64;
      uint16_t* dq = pl->d_jqt + (size_t)sl * kMaxJpegQt * 64;
      const int nset = (int)pl->jset_hdr.size();
      for (int t = 0; t < nset; ++t) {
        const JpegHdr& H = pl->jhdr[pl->jset_hdr[t]];
        for (int cl = 0; cl < 2; ++cl)
          for (int id = 0; id < 4; ++id) {
            HuffTable& T = cl ? hh[t].ac[id] : hh[t].dc[id];
            if (H.ht_ok[cl][id]) build_huff(H.bits[cl][id], H.vals[cl][id], T);
            else empty_huff(T);
          }
      }
      for (size_t t = 0; t < pl->jqt.size(); ++t) memcpy(hq + 64 * t, pl->jqt[t].data(), 128);
      int64_t nseg_total = 0, nact_total = 0;
      int nact_img = 0;
      for (int i = 0; i < n_images; ++i) {
        const JpegHdr& H = pl->jhdr[pl->jimg_hdr[i]];
        const ExpandDesc& e = he[i];
        JpegDesc& J = hj[i];
        J.data = pl->cbuf[sl] + (ji[i].offset - lo);
        J.tabs = dh + pl->jhdr_set[pl->jimg_hdr[i]];
        J.size = (int32_t)ji[i].size;
        J.scan_off = H.scan_off;
        const TileLayout& L = Ls[hr[i].kind];
        for (int c = 0; c < 3; ++c) {
          J.dst[c] = e.dst[c];
          J.dst_stride[c] = e.dst_stride[c];
          J.nbx[c] = c < H.ncomp ? e.nbx[c] : 0;
          J.nby[c] = c < H.ncomp ? e.nby[c] : 0;
          J.bx0[c] = L.bx0[c];
          J.by0[c] = L.by0[c];
          J.h[c] = (uint8_t)H.h[c]; J.v[c] = (uint8_t)H.v[c];
          J.td[c] = (uint8_t)H.td[c]; J.ta[c] = (uint8_t)H.ta[c];
        }
        J.mcus_x = H.mcus_x;
        J.nmcu = H.mcus_x * H.mcus_y;
        J.ri = H.ri > 0 ? H.ri : J.nmcu;
        J.nseg = H.nseg;
        J.seg_base = (int32_t)nseg_total;
        J.E = E;
        J.ncomp = (uint8_t)H.ncomp;
        nseg_total += H.nseg;
        // intervals holding ROI blocks (the decode grid; equal for
        // consecutive images of one header and kind)
        if (!(i > 0 && pl->jimg_hdr[i] == pl->jimg_hdr[i - 1] && hr[i].kind == hr[i - 1].kind)) {
          nact_img = 0;
          for (int sg = 0; sg < J.nseg; ++sg) nact_img += seg_in_roi(J, sg) ? 1 : 0;
        }
        nact_total += nact_img;
      }
      if (nseg_total >= INT_MAX / 2) return fail(SMOL_ERR_CAPACITY, "%lld restart intervals in one batch", (long long)nseg_total);
      void* segb = pl->d_seg[sl];
      rc = grow(&segb, &pl->seg_cap[sl], (size_t)nseg_total * 12 + 16, pl->copy_stream, pl->fixed_stage, "segment index");
      pl->d_seg[sl] = static_cast<int32_t*>(segb);
      if (rc) return rc;
      pl->jnseg = (int)nseg_total;
      pl->jnact = (int)nact_total;
      SMOL_CUDA(cudaMemcpyAsync(dj, hj, sizeof(JpegDesc) * n_images, cudaMemcpyHostToDevice, pl->copy_stream));
      SMOL_CUDA(cudaMemcpyAsync(dh, hh, sizeof(HuffSet) * nset, cudaMemcpyHostToDevice, pl->copy_stream));
      SMOL_CUDA(cudaMemcpyAsync(dq, hq, 128 * pl->jqt.size(), cudaMemcpyHostToDevice, pl->copy_stream));
      SMOL_CUDA(cudaMemcpyAsync(d, h, sizeof(DevImage) * nk, cudaMemcpyHostToDevice, pl->copy_stream));
      SMOL_CUDA(cudaMemcpyAsync(dr, hr, sizeof(DevRef) * n_images, cudaMemcpyHostToDevice, pl->copy_stream));
      if (nl) SMOL_CUDA(cudaMemcpyAsync(dl, hl, sizeof(TileLayout) * nl, cudaMemcpyHostToDevice, pl->copy_stream));
      if (ntap) SMOL_CUDA(cudaMemcpyAsync(dt, ht, sizeof(int4) * ntap, cudaMemcpyHostToDevice, pl->copy_stream));
      SMOL_CUDA(cudaMemcpyAsync(pl->cbuf[sl], arena + lo, (size_t)(hi - lo), cudaMemcpyHostToDevice, pl->copy_stream));
      qtables = dq;
    }
    if (map_n)
      SMOL_CUDA(cudaMemcpyAsync(dm, hm, sizeof(int4) * map_n, cudaMemcpyHostToDevice, pl->copy_stream));
    SMOL_CUDA(cudaEventRecord(pl->stage_ready[sl], pl->copy_stream));
    if (src == Src::kJpeg) {
      // marker index (warp per image) + Huffman decode (thread per restart
      // interval) on the expand stream, into the staged ROI planes
      cudaStream_t es = pl->expand_own_stream ? pl->expand_stream : stream;
      const int sl_ = sl;
      JpegDesc* dj = pl->d_jdesc + (size_t)sl_ * pl->max_images;
      int32_t* seg_start = pl->d_seg[sl_];
      int32_t* seg_img = seg_start + pl->jnseg;
      int32_t* active = seg_img + pl->jnseg;
      int32_t* n_active = active + pl->jnseg;
      SMOL_CUDA(cudaStreamWaitEvent(es, pl->stage_ready[sl_], 0));
      SMOL_CUDA(cudaMemsetAsync(n_active, 0, sizeof(int32_t), es));
      smol_jpeg_index_kernel<<<n_images, 32 * kIndexWarps, 0, es>>>(dj, n_images, seg_start, seg_img, active,
                                                                    n_active);
      SMOL_CUDA(cudaGetLastError());
      smol_jpeg_decode_kernel<<<ceil_div(std::max(pl->jnact, 1), kJpegThreads), kJpegThreads, 0, es>>>(
          dj, pl->jnseg, seg_start, seg_img, active, n_active, pl->d_zmap,
          pl->d_huff + (size_t)sl_ * kMaxHuffSets, pl->jset_hdr.size() == 1 ? 1 : 0);
      SMOL_CUDA(cudaGetLastError());
      if (es != stream) {
        SMOL_CUDA(cudaEventRecord(pl->stage_expanded[sl_], es));
        SMOL_CUDA(cudaStreamWaitEvent(stream, pl->stage_expanded[sl_], 0));
      }
    } else if (src == Src::kCompact) {
      // expand on the plan's expand stream: the copy stream carries only
      // copies (batch k+1's transfer overlaps batch k's kernels) and the
      // expansion of batch k+1 runs in the tail of batch k's fused kernel
      // instead of between the fused kernels on `stream`
      cudaStream_t es = pl->expand_own_stream ? pl->expand_stream : stream;
      SMOL_CUDA(cudaStreamWaitEvent(es, pl->stage_ready[sl], 0));
      smol_expand_kernel<<<n_images * kExpandSplit, kExpandWarps * 32, kExpandSmem, es>>>(de);
      SMOL_CUDA(cudaGetLastError());
      if (es != stream) {
        SMOL_CUDA(cudaEventRecord(pl->stage_expanded[sl], es));
        SMOL_CUDA(cudaStreamWaitEvent(stream, pl->stage_expanded[sl], 0));
      }
    } else {
      SMOL_CUDA(cudaStreamWaitEvent(stream, pl->stage_ready[sl], 0));
    }
  }

  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  SMOL_CUDA(cudaStreamIsCapturing(stream, &cap));
  if (src == Src::kDevice && cap != cudaStreamCaptureStatusNone) {
    // (being captured into a CUDA graph: keep every operation on `stream`)
    SMOL_CUDA(cudaMemcpyAsync(d, h, sizeof(DevImage) * nk, cudaMemcpyHostToDevice, stream));
    SMOL_CUDA(cudaMemcpyAsync(dr, hr, sizeof(DevRef) * n_images, cudaMemcpyHostToDevice, stream));
    if (nl) SMOL_CUDA(cudaMemcpyAsync(dl, hl, sizeof(TileLayout) * nl, cudaMemcpyHostToDevice, stream));
    if (ntap) SMOL_CUDA(cudaMemcpyAsync(dt, ht, sizeof(int4) * ntap, cudaMemcpyHostToDevice, stream));
    if (map_n) SMOL_CUDA(cudaMemcpyAsync(dm, hm, sizeof(int4) * map_n, cudaMemcpyHostToDevice, stream));
  } else if (src == Src::kDevice) {
    // descriptors (and the CTA map) go up on the plan's copy stream, so the
    // copy for run k+1 overlaps run k's kernel instead of sitting between
    // the kernels on `stream` (4096 thumbnails: 512 KB per run); the ring
    // slot is free (host waited on ev[slot] above)
    SMOL_CUDA(cudaMemcpyAsync(d, h, sizeof(DevImage) * nk, cudaMemcpyHostToDevice, pl->copy_stream));
    SMOL_CUDA(cudaMemcpyAsync(dr, hr, sizeof(DevRef) * n_images, cudaMemcpyHostToDevice, pl->copy_stream));
    if (nl) SMOL_CUDA(cudaMemcpyAsync(dl, hl, sizeof(TileLayout) * nl, cudaMemcpyHostToDevice, pl->copy_stream));
    if (ntap) SMOL_CUDA(cudaMemcpyAsync(dt, ht, sizeof(int4) * ntap, cudaMemcpyHostToDevice, pl->copy_stream));
    if (map_n) SMOL_CUDA(cudaMemcpyAsync(dm, hm, sizeof(int4) * map_n, cudaMemcpyHostToDevice, pl->copy_stream));
    SMOL_CUDA(cudaEventRecord(pl->desc_ready[slot], pl->copy_stream));
    SMOL_CUDA(cudaStreamWaitEvent(stream, pl->desc_ready[slot], 0));
  }
  KParams kp = dbg ? *dbg : KParams{};
  kp.refs = dr;
  kp.kinds = d;
  kp.lays = nl ? dl : nullptr;
  kp.lay_stride = lay_stride;
  kp.taps = dt;
  kp.qtables = qtables;
  kp.out = out;
  kp.OW = pl->OW; kp.OH = pl->OH; kp.tile_rows = tile_rows;
  kp.magic = 0x4B000000u;
  kp.out_vec = reinterpret_cast<uintptr_t>(out) % (4 * out_esz) == 0;
  // Row-run output tasks pay off when consecutive output rows share source
  // rows, i.e. under vertical magnification (measured r02: c3b 0.0556 ->
  // 0.0488 ms, c3a 0.0822 -> 0.0800; slower where rows are skipped: c2, c5).
  // Run length by the batch's weakest vertical magnification: 32 rows from
  // 2x (r02t: c3b at 2.7x 0.0370 -> 0.0357 ms), else 8 (c3a at 1.36x: 32
  // rows 0.0757 vs 0.0663 ms).
  double vmag = 1e30;
  for (int i = 0; i < nk; ++i) vmag = std::min(vmag, (double)h[i].Hr / std::max(h[i].sh, 1));
  kp.rowrun = vmag >= 2.0 ? 32 : vmag >= 1.0 ? 8 : 0;
  kp.tile_cols = cols_of(n_col_tiles);
  kp.n_col_tiles = n_col_tiles = ceil_div(pl->OW, kp.tile_cols);
  for (int c = 0; c < 3; ++c) { kp.na[c] = pl->na[c]; kp.nb[c] = pl->nb[c]; }
  kp.cta_map = map_n ? dm : nullptr;
  if (thumb) {
    const bool f16 = pl->p.out_dtype == SMOL_OUT_F16_NCHW;
    auto tk = f16 ? (packed ? smol_thumb_kernel<true, true> : smol_thumb_kernel<true, false>)
                  : (packed ? smol_thumb_kernel<false, true> : smol_thumb_kernel<false, false>);
    const int grid_t = imin(ceil_div(n_images, kThumbWarps), pl->num_sms * 16);
    tk<<<grid_t, kThumbWarps * 32, kThumbSmem, stream>>>(kp, n_images);
    SMOL_CUDA(cudaGetLastError());
    SMOL_CUDA(cudaEventRecord(pl->ev[slot], stream));
    if (sl_used >= 0) SMOL_CUDA(cudaEventRecord(pl->stage_free[sl_used], stream));
    return SMOL_OK;
  }
  kp.n_row_tiles = ntiles;
  const long long nblk = map_n ? (long long)map_n : (long long)ntiles * n_col_tiles * n_images;
  if (nblk >= INT_MAX) return fail(SMOL_ERR_CAPACITY, "%lld CTAs exceed the grid limit", nblk);
  dim3 grid((unsigned)nblk, 1);
  fn<<<grid, cta_threads, smem, stream>>>(kp);
  SMOL_CUDA(cudaGetLastError());
  SMOL_CUDA(cudaEventRecord(pl->ev[slot], stream));
  if (sl_used >= 0) SMOL_CUDA(cudaEventRecord(pl->stage_free[sl_used], stream));
  return SMOL_OK;
}

int32_t run_batch(smol_preproc_plan_t* pl, const smol_batch_desc* b, void* out, void* stream,
                  const KParams* dbg, Src src) {
  g_last_error.clear();
  if (!pl) return fail(SMOL_ERR_INVALID, "plan is NULL");
  if (!b) return fail(SMOL_ERR_INVALID, "batch is NULL");
  return run_impl(pl, b->n_images, b->images, b->qtables, b->n_qtables, out, stream, dbg, src);
}

// Compact record of one image (format: include/smol_preproc.h).  Pass 1
// (dst == NULL) counts, pass 2 writes.
int64_t compact_encode_pass(const smol_image_desc* d, const TileLayout& L, int E, uint64_t mask_y,
                            uint64_t mask_c, uint8_t* dst, uint32_t* n_units_out) {
  int64_t nblocks = 0, nrows = 0;
  for (int c = 0; c < 3; ++c) {
    nblocks += (int64_t)(L.bx1[c] - L.bx0[c] + 1) * (L.by1[c] - L.by0[c] + 1);
    nrows += L.by1[c] - L.by0[c] + 1;
  }
  uint8_t* lens = dst ? dst + kCompactHeader : nullptr;
  uint32_t* rs = dst ? reinterpret_cast<uint32_t*>(dst + compact_rowstart_off(nblocks)) : nullptr;
  uint16_t* units = dst ? reinterpret_cast<uint16_t*>(dst + compact_entries_off(nblocks, nrows)) : nullptr;
  uint32_t nu = 0;
  int64_t bi = 0, ri = 0;
  for (int c = 0; c < 3; ++c) {
    const int stride = d->row_stride_bytes[c] / 2;
    const uint64_t mask = c ? mask_c : mask_y;          // (chroma at twice the scale: its own set)
    for (int by = L.by0[c]; by <= L.by1[c]; ++by) {
      if (rs) rs[ri] = nu;
      ++ri;
      for (int bx = L.bx0[c]; bx <= L.bx1[c]; ++bx) {
        const int16_t* blk = d->coef[c] + (size_t)by * stride + (size_t)bx * E;
        const uint32_t first = nu;
        for (int e = 0; e < E; ++e) {
          const int v = blk[e];
          if (!((mask >> e) & 1) || v == 0) continue;
          if (v >= -511 && v <= 511) {
            if (units) units[nu] = (uint16_t)(e | (v << 6));
            nu += 1;
          } else {
            if (units) { units[nu] = (uint16_t)(e | (kEscape << 6)); units[nu + 1] = (uint16_t)(int16_t)v; }
            nu += 2;
          }
        }
        if (lens) lens[bi] = (uint8_t)(nu - first);          // <= 2 * 64
        ++bi;
      }
    }
  }
  *n_units_out = nu;
  return compact_record_bytes(nblocks, nrows, nu);
}

}  // namespace

extern "C" {

int32_t smol_preproc_run(smol_preproc_plan_t* pl, const smol_batch_desc* b, void* out, void* stream) {
  return run_batch(pl, b, out, stream, nullptr, Src::kDevice);
}

int32_t smol_preproc_run_host(smol_preproc_plan_t* pl, const smol_batch_desc* b, void* out, void* stream) {
  // Pinned host coefficient memory is device-addressable under UVA.  Only the
  // ROI block rows cross PCIe: a gather kernel on the plan's copy stream
  // stages them (3 staging slots, so batch k+1's transfer overlaps batch k's
  // fused kernel while the host prepares batch k+2), then the fused kernel runs on `stream`.
  // Every plane must be pinned host (or device) memory: the gather kernel
  // reads it over PCIe, and a pageable pointer would fault the context.  Each
  // plane's first and last byte is checked, with verified allocations cached
  // (driver range query) so a batch from one pinned arena costs one query.
  if (pl && b && b->images && b->n_images > 0) {
    static CUresult (*get_attr)(void*, CUpointer_attribute, CUdeviceptr) = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
      void* fn = nullptr;
      cudaDriverEntryPointQueryResult q;
      if (cudaGetDriverEntryPoint("cuPointerGetAttribute", &fn, cudaEnableDefault, &q) == cudaSuccess &&
          q == cudaDriverEntryPointSuccess)
        get_attr = reinterpret_cast<CUresult (*)(void*, CUpointer_attribute, CUdeviceptr)>(fn);
    });
    auto usable = [&](uintptr_t a) -> bool {
      for (const auto& r : pl->pinned_ok)
        if (a >= r.first && a < r.second) return true;
      cudaPointerAttributes pa;
      if (cudaPointerGetAttributes(&pa, reinterpret_cast<const void*>(a)) != cudaSuccess ||
          (pa.type != cudaMemoryTypeHost && pa.type != cudaMemoryTypeDevice && pa.type != cudaMemoryTypeManaged)) {
        cudaGetLastError();
        return false;
      }
      CUdeviceptr start = 0;
      size_t size = 0;
      if (get_attr && get_attr(&start, CU_POINTER_ATTRIBUTE_RANGE_START_ADDR, (CUdeviceptr)a) == CUDA_SUCCESS &&
          get_attr(&size, CU_POINTER_ATTRIBUTE_RANGE_SIZE, (CUdeviceptr)a) == CUDA_SUCCESS && size > 0 &&
          a >= (uintptr_t)start && a < (uintptr_t)start + size) {
        // (device pointer range; for pinned host memory mapped at the same
        // address under UVA it is the host range)
        if (pl->pinned_ok.size() >= 64) pl->pinned_ok.erase(pl->pinned_ok.begin());
        pl->pinned_ok.emplace_back((uintptr_t)start, (uintptr_t)start + size);
      }
      return true;
    };
    for (int i = 0; i < b->n_images; ++i) {
      const smol_image_desc& d = b->images[i];
      for (int c = 0; c < (d.subsampling == 400 ? 1 : 3); ++c) {
        const uintptr_t lo = reinterpret_cast<uintptr_t>(d.coef[c]);
        const long long span = (long long)std::max(d.blocks_h[c], 1) * d.row_stride_bytes[c];
        if (!d.coef[c] || span <= 0) continue;          // run_impl reports the descriptor error
        if (!usable(lo) || !usable(lo + (uintptr_t)span - 1))
          return fail(SMOL_ERR_INVALID, "image %d: coef[%d] is neither pinned host nor device memory", i, c);
      }
    }
  }
  return run_batch(pl, b, out, stream, nullptr, Src::kGather);
}

int32_t smol_preproc_run_compact(smol_preproc_plan_t* pl, const smol_compact_batch* b, void* out, void* stream) {
  g_last_error.clear();
  if (!pl) return fail(SMOL_ERR_INVALID, "plan is NULL");
  if (!b) return fail(SMOL_ERR_INVALID, "batch is NULL");
  if (b->n_images > 0 && (!b->arena || reinterpret_cast<uintptr_t>(b->arena) % 16 || b->arena_bytes <= 0))
    return fail(SMOL_ERR_INVALID, "compact arena NULL, not 16-byte aligned or empty");
  return run_impl(pl, b->n_images, b->images, b->qtables, b->n_qtables, out, stream, nullptr, Src::kCompact, b);
}

int32_t smol_jpeg_parse_header(const void* data, int64_t size, smol_jpeg_header* out) {
  g_last_error.clear();
  if (!data || !out) return fail(SMOL_ERR_INVALID, "data/out is NULL");
  JpegHdr H;
  int32_t rc = parse_jpeg(static_cast<const uint8_t*>(data), size, 0, H);
  if (rc) return rc;
  memset(out, 0, sizeof(*out));
  out->width = H.width; out->height = H.height; out->subsampling = H.subsampling; out->ncomp = H.ncomp;
  for (int c = 0; c < 3; ++c) { out->blocks_w[c] = H.blocks_w[c]; out->blocks_h[c] = H.blocks_h[c]; }
  out->mcus_x = H.mcus_x; out->mcus_y = H.mcus_y;
  out->restart_interval = H.ri;
  out->n_segments = H.nseg;
  out->scan_offset = H.scan_off;
  return SMOL_OK;
}

namespace {
// Batch checks shared by run_jpeg and decode_planes: host-readable arena,
// files inside it.
int32_t check_jpeg_batch(const smol_jpeg_batch* b) {
  if (!b) return fail(SMOL_ERR_INVALID, "batch is NULL");
  if (b->n_images < 0) return fail(SMOL_ERR_INVALID, "n_images=%d < 0", b->n_images);
  if (b->n_images == 0) return SMOL_OK;
  if (!b->images || !b->arena || b->arena_bytes <= 0) return fail(SMOL_ERR_INVALID, "images/arena NULL or empty");
  cudaPointerAttributes pa;
  if (cudaPointerGetAttributes(&pa, b->arena) != cudaSuccess || pa.type != cudaMemoryTypeHost) {
    cudaGetLastError();
    return fail(SMOL_ERR_INVALID, "JPEG arena must be pinned host memory (headers are parsed on the host)");
  }
  for (int i = 0; i < b->n_images; ++i) {
    const smol_jpeg_image& m = b->images[i];
    if (m.offset < 0 || m.offset % 16 || m.size < 4 || m.offset + m.size > b->arena_bytes || m.size > INT_MAX)
      return fail(SMOL_ERR_INVALID, "image %d: file [%lld, +%lld) not 16-B aligned or outside the arena of %lld B", i,
                  (long long)m.offset, (long long)m.size, (long long)b->arena_bytes);
  }
  return SMOL_OK;
}

// Distinct headers of a batch (an image whose header bytes equal the previous
// image's reuses its parse), their quantization tables and table sets.
int32_t parse_jpeg_batch(smol_preproc_plan_t* pl, const smol_jpeg_batch* b) {
  const uint8_t* arena = static_cast<const uint8_t*>(b->arena);
  const int n = b->n_images;
  pl->jhdr.clear(); pl->jhdr_set.clear(); pl->jset_hdr.clear(); pl->jqt.clear(); pl->jhdr_qid.clear();
  pl->jimg_hdr.resize(n);
  pl->jci.resize(n);
  for (int i = 0; i < n; ++i) {
    const smol_jpeg_image& m = b->images[i];
    const uint8_t* data = arena + m.offset;
    bool same = false;
    if (i > 0) {
      const JpegHdr& P = pl->jhdr[pl->jimg_hdr[i - 1]];
      const uint8_t* pd = arena + b->images[i - 1].offset;
      same = m.size > P.scan_off && memcmp(data, pd, (size_t)P.scan_off) == 0;
    }
    if (same) {
      pl->jimg_hdr[i] = pl->jimg_hdr[i - 1];
    } else {
      pl->jhdr.emplace_back();
      JpegHdr& H = pl->jhdr.back();
      int32_t rc = parse_jpeg(data, m.size, i, H);
      if (rc) return rc;
      std::array<int, 3> qid{0, 0, 0};
      for (int c = 0; c < H.ncomp; ++c) {
        std::array<uint16_t, 64> q;
        memcpy(q.data(), H.qt[H.tq[c]], 128);
        int k = 0;
        while (k < (int)pl->jqt.size() && pl->jqt[k] != q) ++k;
        if (k == (int)pl->jqt.size()) {
          if (k >= kMaxJpegQt) return fail(SMOL_ERR_CAPACITY, "more than %d distinct quantization tables", kMaxJpegQt);
          pl->jqt.push_back(q);
        }
        qid[c] = k;
      }
      pl->jhdr_qid.push_back(qid);
      int t = 0;
      for (; t < (int)pl->jset_hdr.size(); ++t) {
        const JpegHdr& O = pl->jhdr[pl->jset_hdr[t]];
        if (!memcmp(O.ht_ok, H.ht_ok, sizeof(H.ht_ok)) && !memcmp(O.bits, H.bits, sizeof(H.bits)) &&
            !memcmp(O.vals, H.vals, sizeof(H.vals)))
          break;
      }
      if (t == (int)pl->jset_hdr.size()) {
        if (t >= kMaxHuffSets) return fail(SMOL_ERR_CAPACITY, "more than %d distinct Huffman table sets", kMaxHuffSets);
        pl->jset_hdr.push_back((int)pl->jhdr.size() - 1);
      }
      pl->jhdr_set.push_back(t);
      pl->jimg_hdr[i] = (int)pl->jhdr.size() - 1;
    }
    const int hi = pl->jimg_hdr[i];
    const JpegHdr& H = pl->jhdr[hi];
    smol_compact_image& ci = pl->jci[i];
    memset(&ci, 0, sizeof(ci));
    ci.width = H.width; ci.height = H.height; ci.subsampling = H.subsampling;
    for (int c = 0; c < 3; ++c) ci.qtable[c] = c < H.ncomp ? pl->jhdr_qid[hi][c] : 0;
    ci.roi_left = m.roi_left; ci.roi_top = m.roi_top;
    ci.roi_x = m.roi_x; ci.roi_y = m.roi_y; ci.roi_w = m.roi_w; ci.roi_h = m.roi_h;
    ci.offset = 0;
  }
  return SMOL_OK;
}
}  // namespace

int32_t smol_preproc_run_jpeg(smol_preproc_plan_t* pl, const smol_jpeg_batch* b, void* out, void* stream) {
  g_last_error.clear();
  if (!pl) return fail(SMOL_ERR_INVALID, "plan is NULL");
  int32_t rc = check_jpeg_batch(b);
  if (rc || b->n_images == 0) return rc;
  if (b->n_images > pl->max_images)
    return fail(SMOL_ERR_CAPACITY, "n_images=%d > plan capacity %d", b->n_images, pl->max_images);
  if (pl->p.chroma_2s) return fail(SMOL_ERR_UNSUPPORTED, "run_jpeg with chroma_2s plans");
  rc = parse_jpeg_batch(pl, b);
  if (rc) return rc;
  return run_impl(pl, b->n_images, pl->jci.data(), nullptr, (int)pl->jqt.size(), out, stream, nullptr, Src::kJpeg,
                  nullptr, b);
}

int32_t smol_jpeg_decode_planes(const smol_jpeg_batch* b, int16_t* const* planes, void* stream_v) {
  g_last_error.clear();
  int32_t rc = check_jpeg_batch(b);
  if (rc || b->n_images == 0) return rc;
  if (!planes) return fail(SMOL_ERR_INVALID, "planes is NULL");
  cudaStream_t stream = reinterpret_cast<cudaStream_t>(stream_v);
  const int n = b->n_images;
  std::vector<JpegHdr> hs(n);
  std::vector<JpegDesc> js(n);
  std::vector<HuffSet> sets(n);
  int64_t lo = INT64_MAX, hi = 0, nseg = 0;
  for (int i = 0; i < n; ++i) {
    const smol_jpeg_image& m = b->images[i];
    rc = parse_jpeg(static_cast<const uint8_t*>(b->arena) + m.offset, m.size, i, hs[i]);
    if (rc) return rc;
    lo = std::min<int64_t>(lo, m.offset);
    hi = std::max<int64_t>(hi, m.offset + m.size);
    nseg += hs[i].nseg;
  }
  const std::array<int, 64> zz = zigzag_order();
  int8_t zm[64];
  for (int k = 0; k < 64; ++k) zm[k] = (int8_t)zz[k];
  uint8_t* dd = nullptr;
  JpegDesc* dj = nullptr;
  HuffSet* dh = nullptr;
  int32_t* dseg = nullptr;
  int8_t* dz = nullptr;
  auto cleanup = [&] {
    if (dd) cudaFree(dd);
    if (dj) cudaFree(dj);
    if (dh) cudaFree(dh);
    if (dseg) cudaFree(dseg);
    if (dz) cudaFree(dz);
  };
  cudaError_t e = cudaMalloc(&dd, (size_t)(hi - lo) + 16);     // (the bit reader's 4-byte loads may read 7 B ahead)
  if (e == cudaSuccess) e = cudaMalloc(&dj, sizeof(JpegDesc) * n);
  if (e == cudaSuccess) e = cudaMalloc(&dh, sizeof(HuffSet) * n);
  if (e == cudaSuccess) e = cudaMalloc(&dseg, 12 * (size_t)nseg + 16);
  if (e == cudaSuccess) e = cudaMalloc(&dz, 64);
  nseg = 0;
  for (int i = 0; i < n && e == cudaSuccess; ++i) {
    const JpegHdr& H = hs[i];
    for (int cl = 0; cl < 2; ++cl)
      for (int id = 0; id < 4; ++id) {
        HuffTable& T = cl ? sets[i].ac[id] : sets[i].dc[id];
        if (H.ht_ok[cl][id]) build_huff(H.bits[cl][id], H.vals[cl][id], T);
        else empty_huff(T);
      }
    JpegDesc& J = js[i];
    memset(&J, 0, sizeof(J));
    J.data = dd + (b->images[i].offset - lo);
    J.tabs = dh + i;
    J.size = (int32_t)b->images[i].size;
    J.scan_off = H.scan_off;
    for (int c = 0; c < H.ncomp; ++c) {
      J.dst[c] = planes[3 * i + c];
      if (!J.dst[c]) { e = cudaErrorInvalidValue; break; }
      J.dst_stride[c] = H.blocks_w[c] * 64;
      J.nbx[c] = H.blocks_w[c];
      J.nby[c] = H.blocks_h[c];
      J.h[c] = (uint8_t)H.h[c]; J.v[c] = (uint8_t)H.v[c];
      J.td[c] = (uint8_t)H.td[c]; J.ta[c] = (uint8_t)H.ta[c];
    }
    J.mcus_x = H.mcus_x;
    J.nmcu = H.mcus_x * H.mcus_y;
    J.ri = H.ri > 0 ? H.ri : J.nmcu;
    J.nseg = H.nseg;
    J.seg_base = (int32_t)nseg;
    J.E = 64;
    J.ncomp = (uint8_t)H.ncomp;
    nseg += H.nseg;
  }
  if (e == cudaSuccess) e = cudaMemcpyAsync(dd, static_cast<const uint8_t*>(b->arena) + lo, (size_t)(hi - lo),
                                            cudaMemcpyHostToDevice, stream);
  if (e == cudaSuccess) e = cudaMemcpyAsync(dj, js.data(), sizeof(JpegDesc) * n, cudaMemcpyHostToDevice, stream);
  if (e == cudaSuccess) e = cudaMemcpyAsync(dh, sets.data(), sizeof(HuffSet) * n, cudaMemcpyHostToDevice, stream);
  if (e == cudaSuccess) e = cudaMemcpyAsync(dz, zm, 64, cudaMemcpyHostToDevice, stream);
  if (e == cudaSuccess) e = cudaMemsetAsync(dseg + 3 * nseg, 0, sizeof(int32_t), stream);
  if (e == cudaSuccess) {
    smol_jpeg_index_kernel<<<n, 32 * kIndexWarps, 0, stream>>>(dj, n, dseg, dseg + nseg, dseg + 2 * nseg,
                                                                dseg + 3 * nseg);
    smol_jpeg_decode_kernel<<<(int)((nseg + kJpegThreads - 1) / kJpegThreads), kJpegThreads, 0, stream>>>(
        dj, (int)nseg, dseg, dseg + nseg, dseg + 2 * nseg, dseg + 3 * nseg, dz, dh, 0);
    e = cudaGetLastError();
  }
  if (e == cudaSuccess) e = cudaStreamSynchronize(stream);
  cleanup();
  if (e != cudaSuccess) return fail(SMOL_ERR_CUDA, "jpeg decode: %s", cudaGetErrorString(e));
  return SMOL_OK;
}

int32_t smol_compact_encode(const smol_preproc_params* p, const smol_image_desc* d, void* dst, int64_t capacity,
                            int64_t* written) {
  g_last_error.clear();
  int32_t rc = validate_params(p);
  if (rc) return rc;
  if (!d || !written) return fail(SMOL_ERR_INVALID, "image/written is NULL");
  DevImage g{};
  rc = validate_image(p, d, 0, 4, g, /*need_align=*/false);
  if (rc) return rc;
  const int OW = p->crop_w > 0 ? p->crop_w : g.Wr, OH = p->crop_w > 0 ? p->crop_h : g.Hr;
  TileLayout L;
  tile_layout(g, p->scale_denom, 0, OH, 0, OW, L, kYPWide, true);
  const int E = block_elems(p->scale_denom, p->layout, p->idct_def);
  const uint64_t mask = used_mask(p->scale_denom, p->layout == SMOL_LAYOUT_PACKED, p->idct_def == SMOL_IDCT_TRUNCATED);
  const uint64_t mask_c = used_mask(g.ck, p->layout == SMOL_LAYOUT_PACKED, p->idct_def == SMOL_IDCT_TRUNCATED);
  uint32_t nv = 0;
  const int64_t bytes = compact_encode_pass(d, L, E, mask, mask_c, nullptr, &nv);
  *written = bytes;
  if (!dst) return SMOL_OK;
  if (capacity < bytes)
    return fail(SMOL_ERR_CAPACITY, "compact record needs %lld B > capacity %lld", (long long)bytes,
                (long long)capacity);
  uint8_t* o = static_cast<uint8_t*>(dst);
  memset(o, 0, (size_t)bytes);
  CompactHeader hd{};
  hd.magic = kCompactMagic;
  hd.E = (uint32_t)E;
  hd.n_units = nv;
  for (int c = 0; c < 3; ++c) {
    hd.bx0[c] = L.bx0[c]; hd.by0[c] = L.by0[c];
    hd.nbx[c] = L.bx1[c] - L.bx0[c] + 1; hd.nby[c] = L.by1[c] - L.by0[c] + 1;
  }
  memcpy(o, &hd, sizeof(hd));
  compact_encode_pass(d, L, E, mask, mask_c, o, &nv);
  return SMOL_OK;
}

int32_t smol_debug_run(smol_preproc_plan_t* pl, const smol_batch_desc* b, void* out, int16_t* y_dbg,
                       int16_t* cb_dbg, int16_t* cr_dbg, int16_t* rgb_dbg, int64_t sy, int64_t sc,
                       int64_t srgb, void* stream) {
  if (!y_dbg || !cb_dbg || !cr_dbg || !rgb_dbg) return fail(SMOL_ERR_INVALID, "debug buffer is NULL");
  KParams kp{};
  kp.dbg_pl[0] = y_dbg; kp.dbg_pl[1] = cb_dbg; kp.dbg_pl[2] = cr_dbg; kp.dbg_rgb = rgb_dbg;
  kp.dbg_stride_y = sy; kp.dbg_stride_c = sc; kp.dbg_stride_rgb = srgb;
  return run_batch(pl, b, out, stream, &kp, Src::kDevice);
}

}  // extern "C"
