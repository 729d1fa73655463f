// smol_jpeg.cuh -- GPU entropy decoding of baseline JPEG:
// restart-interval parallelism.  The paper keeps Huffman decoding on the host
// because it "requires substantial branching" (§6.4); here the
// host only parses the headers (markers, tables: a few hundred bytes per
// distinct header), and two kernels do the per-byte work:
//   1. smol_jpeg_index_kernel  (warp per image): find the RSTm markers in the
//      entropy-coded data (T.81 B.2.1, E.1.4) -> first byte of every restart
//      interval ("segment");
//   2. smol_jpeg_decode_kernel (thread per segment): Huffman-decode the
//      segment's MCUs (T.81 F.2.2: DC difference with a predictor reset at the
//      interval start, F.2.1.3.1; run-length AC with ZRL / EOB, Figure F.13;
//      zig-zag order, Figure A.6) and write the blocks that fall inside the
//      plan's ROI box straight into the staged planes of the plan's layout
//      (dense-64 or packed-for-scale), which the fused kernel then reads as on
//      the compact path.  Segments with no block inside the ROI are skipped:
//      an interval is independently decodable.
// Decoding: one flat loop, one symbol per iteration (DC or AC, any block), so
// a warp's lanes stay on one code path; a 9-bit lookup (length, symbol) for
// short codes, the T.81 F.16 MAXCODE walk for longer ones; a 64-bit bit
// buffer refilled 4 raw bytes at a time when they hold no 0xFF, else byte by
// byte with 0xFF00 unstuffing (B.1.1.5); at a marker the reader feeds zero
// bits (well-formed data never needs them).
#pragma once
#include <stdint.h>

#include "smol_geom.cuh"

namespace smol {

constexpr int kHuffLutBits = 9;

// One Huffman table in the decoder's format (built on the host from a DHT);
// 16-B aligned so the LUT can be copied to shared memory with 16-B loads.
struct alignas(16) HuffTable {
  uint16_t lut[1 << kHuffLutBits];   // code prefix -> length << 8 | symbol (length 0: longer code)
  uint32_t limit[17];                // per length l: codes of length <= l, left-justified to 16 bits, lie
                                     // below limit[l] (canonical codes, T.81 C.2); no code: window >= limit[16]
  int32_t valoff[17];                // per length l: index of HUFFVAL for code c = c + valoff[l]
  uint8_t huffval[256];
};
// The tables of one distinct header: DC and AC, ids 0..3 (T.81 B.2.4.2 Th).
struct HuffSet {
  HuffTable dc[4], ac[4];
};

// One image of a JPEG batch (device descriptor).
struct JpegDesc {
  const uint8_t* data;       // device copy of the file (SOI..EOI)
  int16_t* dst[3];           // staged element (ROI row by0, element bx0 * E) per component
  const HuffSet* tabs;
  int32_t size, scan_off;    // file bytes; first byte of the entropy-coded data
  int32_t dst_stride[3];     // int16 elements per staged row
  int32_t bx0[3], by0[3], nbx[3], nby[3];   // ROI box in blocks per component
  int32_t mcus_x, nmcu, ri, nseg, seg_base; // MCU grid, MCUs per restart interval, segments
  int32_t E;                 // elements per stored block
  uint8_t ncomp, pad0;
  uint8_t h[3], v[3], td[3], ta[3];         // sampling factors, DC/AC table ids
};

#if defined(__CUDACC__)
#ifndef SMOL_JPEG_THREADS
#define SMOL_JPEG_THREADS 128
#endif
#ifndef SMOL_JPEG_SLUT
#define SMOL_JPEG_SLUT 1     // 9-bit LUTs of a single table set in shared memory
#endif
constexpr int kJpegThreads = SMOL_JPEG_THREADS;   // decode CTA size
constexpr int kJpegBlkStride = 72;   // int16 per thread block buffer (144 B: 16-B aligned for 16-byte copies)

// Does restart interval s of image d hold a block inside the ROI box?
// (host: the decode grid is sized from the count)
__host__ __device__ __forceinline__ bool seg_in_roi(const JpegDesc& d, int s) {
  const int m0 = s * d.ri, m1 = (d.nmcu < m0 + d.ri ? d.nmcu : m0 + d.ri) - 1;
  if (m1 < m0) return false;
  const int my0 = m0 / d.mcus_x, my1 = m1 / d.mcus_x;
  const int mxa = my0 == my1 ? m0 - my0 * d.mcus_x : 0;
  const int mxb = my0 == my1 ? m1 - my1 * d.mcus_x : d.mcus_x - 1;
  bool any = false;
  for (int c = 0; c < d.ncomp; ++c) {
    const int H = d.ncomp == 1 ? 1 : d.h[c], V = d.ncomp == 1 ? 1 : d.v[c];
    const int r0 = my0 * V, r1 = my1 * V + V - 1, c0 = mxa * H, c1 = mxb * H + H - 1;
    any |= r0 <= d.by0[c] + d.nby[c] - 1 && r1 >= d.by0[c] && c0 <= d.bx0[c] + d.nbx[c] - 1 && c1 >= d.bx0[c];
  }
  return any;
}

// RST markers (0xFF then 0xD0..0xD7) at positions [clo, chi) of one file,
// by one warp: 512 B per step (16-byte loads; files are 16-B aligned), four
// steps in flight; a marker's second byte may sit in the next lane's (or
// step's) first byte.  Counts them; with `write`, the idx-th marker of the
// scan (idx from `first`) starts segment idx: seg_start[idx] = position + 2.
// 4 warps per image at <= 32 registers (16 CTAs / SM): an index CTA fits
// beside the fused kernel's four CTAs, so batch k+1's marker scan overlaps
// batch k's fused kernel (r02bb: JPEG e2e 0.241-0.254 -> 0.223 ms; 8 warps
// at 64 registers did not fit)
#ifndef SMOL_INDEX_WARPS
#define SMOL_INDEX_WARPS 4
#endif
#ifndef SMOL_INDEX_UNROLL
#define SMOL_INDEX_UNROLL 2
#endif
#ifndef SMOL_INDEX_MINB
#define SMOL_INDEX_MINB 16
#endif
constexpr int kIndexUnroll = SMOL_INDEX_UNROLL, kIndexWarps = SMOL_INDEX_WARPS;
__device__ __forceinline__ int scan_markers(const uint8_t* p, int clo, int chi, int s0, int end, int lane,
                                            bool write, int first, int nseg, int32_t* seg_start) {
  int found = 0;                                  // markers seen so far (whole warp)
  for (int o = clo; o < chi; o += 512 * kIndexUnroll) {
    uint4 w[kIndexUnroll];
#pragma unroll
    for (int u = 0; u < kIndexUnroll; ++u) {
      const int q = o + 512 * u + 16 * lane;
      w[u] = q + 16 <= end ? __ldg(reinterpret_cast<const uint4*>(p + q)) : make_uint4(0, 0, 0, 0);
      if (q < end && q + 16 > end) {              // the file's last partial 16 bytes
        uint32_t t[4] = {0, 0, 0, 0};
        for (int j = 0; j < end - q; ++j) t[j >> 2] |= (uint32_t)__ldg(p + q + j) << (8 * (j & 3));
        w[u] = make_uint4(t[0], t[1], t[2], t[3]);
      }
    }
#pragma unroll
    for (int u = 0; u < kIndexUnroll; ++u) {
      const int q = o + 512 * u + 16 * lane;
      // first byte after this lane's 16: the next lane's first, or the next step's
      // (u is a compile-time constant: every shuffle is executed by the whole warp)
      uint32_t nxt = __shfl_down_sync(0xffffffffu, w[u].x & 0xFFu, 1);
      const uint32_t nstep =
          u + 1 < kIndexUnroll ? (__shfl_sync(0xffffffffu, w[(u + 1) % kIndexUnroll].x, 0) & 0xFFu) : 0u;
      if (lane == 31) nxt = u + 1 < kIndexUnroll ? nstep : (q + 16 < end ? (uint32_t)__ldg(p + q + 16) : 0u);
      // bit j: 0xFF at byte j and 0xD0..0xD7 at byte j + 1, inside [max(clo, s0), chi)
      const uint32_t wd[5] = {w[u].x, w[u].y, w[u].z, w[u].w, nxt};
      uint32_t hits = 0;
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const uint32_t b0 = (wd[j >> 2] >> (8 * (j & 3))) & 0xFFu;
        const uint32_t b1 = j == 15 ? nxt : (wd[(j + 1) >> 2] >> (8 * ((j + 1) & 3))) & 0xFFu;
        if (b0 == 0xFFu && (b1 & 0xF8u) == 0xD0u && q + j >= s0 && q + j < chi && q + j + 1 < end) hits |= 1u << j;
      }
      const int cnt = __popc(hits);
      int inc = cnt;                              // inclusive warp scan of the counts
#pragma unroll
      for (int k = 1; k < 32; k <<= 1) {
        const int t = __shfl_up_sync(0xffffffffu, inc, k);
        if (lane >= k) inc += t;
      }
      if (write) {
        int idx = first + found + inc - cnt;      // markers before this lane's first hit
        while (hits) {
          const int j = __ffs(hits) - 1;
          hits &= hits - 1;
          ++idx;                                  // the idx-th marker starts segment idx
          if (idx < nseg) seg_start[idx] = q + j + 2;
        }
      }
      found += __shfl_sync(0xffffffffu, inc, 31);
    }
  }
  return found;
}

// CTA of kIndexWarps warps per image: segment s > 0 starts after the s-th RST
// marker.  The scan is split into contiguous chunks, one per warp: each warp
// counts its chunk's markers, a CTA prefix gives each chunk its first index,
// then each warp rescans its chunk (L1 / L2 hits) writing the starts.  Also
// appends the image's intervals that hold ROI blocks to the batch's active
// list (the decode kernel's work: no lane idles on a skipped interval).
__global__ void __launch_bounds__(32 * kIndexWarps, SMOL_INDEX_MINB) smol_jpeg_index_kernel(const JpegDesc* ds, int n_images,
                                                                         int32_t* seg_start, int32_t* seg_img,
                                                                         int32_t* active, int32_t* n_active) {
  __shared__ int cnt_s[kIndexWarps];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int img = blockIdx.x;
  if (img >= n_images) return;
  const JpegDesc& d = ds[img];
  const uint8_t* p = d.data;
  const int end = d.size, s0 = d.scan_off;
  const int base = d.seg_base, nseg = d.nseg;
  // defaults (segment 0 at the scan start, missing markers -> empty
  // segments) and the image's intervals holding ROI blocks: counted per
  // thread, one global atomic per CTA, then written at the CTA's offset
  __shared__ int act_s[32 * kIndexWarps];
  __shared__ int act_base;
  int na = 0;
  for (int s = threadIdx.x; s < nseg; s += 32 * kIndexWarps) {
    seg_img[base + s] = img;
    seg_start[base + s] = s == 0 ? s0 : end;
    na += seg_in_roi(d, s) ? 1 : 0;
  }
  act_s[threadIdx.x] = na;
  __syncthreads();
  if (threadIdx.x == 0) {                         // exclusive scan of the counts (256 values)
    int acc = 0;
    for (int i = 0; i < 32 * kIndexWarps; ++i) { const int t = act_s[i]; act_s[i] = acc; acc += t; }
    act_base = acc ? atomicAdd(n_active, acc) : 0;
  }
  __syncthreads();
  int at = act_base + act_s[threadIdx.x];
  if (na)
    for (int s = threadIdx.x; s < nseg; s += 32 * kIndexWarps)
      if (seg_in_roi(d, s)) active[at++] = base + s;
  if (nseg <= 1) return;                          // (uniform over the CTA)
  const int a0 = s0 & ~15;
  const int span = end - a0;
  const int L = ((span + kIndexWarps - 1) / kIndexWarps + 512 * kIndexUnroll - 1) / (512 * kIndexUnroll) *
                (512 * kIndexUnroll);             // chunk: whole steps
  const int clo = min(end, a0 + warp * L), chi = min(end, clo + L);
  const int n = scan_markers(p, clo, chi, s0, end, lane, false, 0, nseg, nullptr);
  if (lane == 0) cnt_s[warp] = n;
  __syncthreads();                                // (after the segment defaults above, too)
  int first = 0;
  for (int w = 0; w < warp; ++w) first += cnt_s[w];
  if (n > 0 && first < nseg - 1) scan_markers(p, clo, chi, s0, end, lane, true, first, nseg, seg_start + base);
}

struct BitReader {
  const uint8_t* p;
  const uint8_t* pend;
  uint64_t buf;              // left-aligned: next bit is bit 63
  int nb;                    // valid bits in buf
  bool stop;                 // met a marker / the end: feed zeros

  // one raw byte with 0xFF00 unstuffing (B.1.1.5); a marker or the end stops
  __device__ __forceinline__ void put_byte() {
    uint32_t b = 0;
    if (!stop) {
      if (p < pend) {
        b = __ldg(p);
        ++p;
        if (b == 0xFFu) {
          const uint32_t b2 = p < pend ? __ldg(p) : 0xD9u;
          if (b2 == 0u) ++p;                      // stuffed 0xFF00
          else { stop = true; b = 0; }            // a marker ends the interval
        }
      } else {
        stop = true;
      }
    }
    buf |= (uint64_t)b << (56 - nb);
    nb += 8;
  }
  // >= 33 valid bits afterwards (one code of <= 16 bits + <= 16 extra bits).
  // Fast path: the next 4 raw bytes (two aligned 32-bit loads, funnel-shifted)
  // hold no 0xFF: append them at once; else byte by byte.
  __device__ __forceinline__ void refill() {
    if (nb > 32) return;
    if (stop) { nb = 64; return; }                // past a marker: the buffer's low bits are already zeros
    if (p + 4 <= pend) {
      const uintptr_t a = reinterpret_cast<uintptr_t>(p);
      const uint32_t* w = reinterpret_cast<const uint32_t*>(a & ~(uintptr_t)3);
      const uint32_t lo = __ldg(w), hi = __ldg(w + 1);
      const uint32_t x = __funnelshift_r(lo, hi, 8 * (uint32_t)(a & 3));   // bytes p..p+3, p in the low byte
      const uint32_t nx = ~x;
      if (((nx - 0x01010101u) & ~nx & 0x80808080u) == 0u) {    // no 0xFF byte
        buf |= (uint64_t)__byte_perm(x, 0u, 0x0123) << (32 - nb);
        nb += 32;
        p += 4;
        return;
      }
    }
    while (nb <= 56) put_byte();
  }
  __device__ __forceinline__ uint32_t peek16() const { return (uint32_t)(buf >> 48); }
  __device__ __forceinline__ void skip(int n) { buf <<= n; nb -= n; }
  // T.81 F.17 RECEIVE + F.12 EXTEND of s <= 16 bits
  __device__ __forceinline__ int32_t receive_extend(int s) {
    if (s == 0) return 0;
    const int32_t v = (int32_t)(buf >> (64 - s));
    skip(s);
    return v < (1 << (s - 1)) ? v - (1 << s) + 1 : v;
  }
};

// T.81 F.16 DECODE (needs >= 16 valid bits): codes of <= 9 bits by one LUT
// read, longer ones by the MAXCODE walk on left-justified limits (a short
// divergent loop; the branch-free form measured slower, r02h)
__device__ __forceinline__ int huff_decode(BitReader& br, const HuffTable* t, const uint16_t* slut = nullptr) {
  const uint32_t look = br.peek16();
  const uint32_t e = slut ? slut[look >> (16 - kHuffLutBits)] : __ldg(&t->lut[look >> (16 - kHuffLutBits)]);
  if (e >> 8) {
    br.skip((int)(e >> 8));
    return (int)(e & 255u);
  }
  int l = kHuffLutBits + 1;
  while (l <= 16 && look >= __ldg(&t->limit[l])) ++l;
  if (l > 16) { br.skip(16); return 0; }        // invalid code: read as EOB / zero
  br.skip(l);
  return (int)__ldg(&t->huffval[((int32_t)(look >> (16 - l)) + __ldg(&t->valoff[l])) & 255]);
}

// Thread per restart interval.  The decode is one flat loop, one symbol per
// iteration whatever the lane's state (DC or AC, any block), so the lanes of
// a warp stay converged on the same code path; a block that ends stores its
// coefficients (if inside the ROI box) and the lane moves to its next block
// (warp-cooperative stores measured slower, r02h).
// one_set: every image of the batch uses table set `set0`, whose 9-bit LUTs
// of tables 0 and 1 are then read from shared memory.
__global__ void __launch_bounds__(kJpegThreads) smol_jpeg_decode_kernel(const JpegDesc* ds, int nseg_total,
                                                                        const int32_t* seg_start,
                                                                        const int32_t* seg_img,
                                                                        const int32_t* active,
                                                                        const int32_t* n_active,
                                                                        const int8_t* dst_index,
                                                                        const HuffSet* set0, int one_set) {
  __shared__ __align__(16) int16_t blkbuf[kJpegThreads * kJpegBlkStride];
#if SMOL_JPEG_SLUT
  __shared__ __align__(16) uint16_t slut[4][1 << kHuffLutBits];   // DC0, DC1, AC0, AC1 of set0
#else
  uint16_t (*slut)[1 << kHuffLutBits] = nullptr;
  one_set = 0;
#endif
  __shared__ uint8_t zmap[64];                    // zig-zag position -> stored element (255: dropped)
  if (threadIdx.x < 64) zmap[threadIdx.x] = (uint8_t)dst_index[threadIdx.x];
  if (one_set) {
    for (int i = threadIdx.x; i < 4 * (1 << kHuffLutBits) / 8; i += kJpegThreads) {
      const int t = i / ((1 << kHuffLutBits) / 8), w = i % ((1 << kHuffLutBits) / 8);
      const HuffTable& T = t == 0 ? set0->dc[0] : t == 1 ? set0->dc[1] : t == 2 ? set0->ac[0] : set0->ac[1];
      reinterpret_cast<uint4*>(slut[t])[w] = __ldg(reinterpret_cast<const uint4*>(T.lut) + w);
    }
  }
  int16_t* blk = blkbuf + threadIdx.x * kJpegBlkStride;
#pragma unroll
  for (int i = 0; i < 8; ++i) reinterpret_cast<uint4*>(blk)[i] = make_uint4(0u, 0u, 0u, 0u);   // (16-B aligned buffers)
  __syncthreads();
  const int gi = blockIdx.x * kJpegThreads + threadIdx.x;
  if (gi >= min(nseg_total, __ldg(n_active))) return;
  const int g = __ldg(active + gi);               // an interval holding ROI blocks
  const JpegDesc& d = ds[seg_img[g]];
  const int s = g - d.seg_base;
  const int m0 = s * d.ri, m1 = min(d.nmcu, m0 + d.ri) - 1;
  const int nc = d.ncomp;
  BitReader br;
  br.p = d.data + seg_start[g];
  br.pend = d.data + d.size;
  br.buf = 0;
  br.nb = 0;
  br.stop = false;
  const int E = d.E;                              // (uniform over a batch)
  // block cursor: MCU (my, mx), component c, block (y, x) inside the MCU
  int my = m0 / d.mcus_x, mx = m0 - my * d.mcus_x, m = m0;
  int c = 0, y = 0, x = 0;
  int H = nc == 1 ? 1 : d.h[0], V = nc == 1 ? 1 : d.v[0];
  const HuffTable* tdc = &d.tabs->dc[d.td[0]];
  const HuffTable* tac = &d.tabs->ac[d.ta[0]];
  // shared-memory LUT rows of the current component's tables (-1: global)
  int sdc = one_set && d.td[0] < 2 ? d.td[0] : -1, sac = one_set && d.ta[0] < 2 ? 2 + d.ta[0] : -1;
  int32_t pred0 = 0, pred1 = 0, pred2 = 0;        // DC predictors (reset per interval, F.2.1.3.1)
  int k = 0;                                      // zig-zag position of the next coefficient
  while (true) {
    br.refill();
    // one symbol: the DC category (k == 0, F.2.2.1) or an AC run/size (F.13)
    const int sl = k == 0 ? sdc : sac;
    const int sym = huff_decode(br, k == 0 ? tdc : tac, sl >= 0 ? slut[sl] : nullptr);
    const int ssss = sym & 15, r = k == 0 ? 0 : sym >> 4;
    if (ssss == 0 && k > 0) {
      k = r == 15 ? k + 16 : 64;                  // ZRL / EOB
    } else {
      k += r;
      int32_t v = br.receive_extend(ssss);
      if (k == 0) {
        const int32_t pv = c == 0 ? pred0 : c == 1 ? pred1 : pred2;
        v += pv;
        if (c == 0) pred0 = v; else if (c == 1) pred1 = v; else pred2 = v;
      }
      if (k < 64) {
        const int e = zmap[k];
        if (e != 255) blk[e] = (int16_t)v;
      }
      ++k;
    }
    if (k < 64) continue;
    // ---- block done: store it if inside the ROI box, clear, next block ----
    {
      const int by = my * V + y - (c == 0 ? d.by0[0] : c == 1 ? d.by0[1] : d.by0[2]);
      const int bx = mx * H + x - (c == 0 ? d.bx0[0] : c == 1 ? d.bx0[1] : d.bx0[2]);
      const int nby = c == 0 ? d.nby[0] : c == 1 ? d.nby[1] : d.nby[2];
      const int nbx = c == 0 ? d.nbx[0] : c == 1 ? d.nbx[1] : d.nbx[2];
      if (by >= 0 && by < nby && bx >= 0 && bx < nbx) {
        int16_t* out = (c == 0 ? d.dst[0] : c == 1 ? d.dst[1] : d.dst[2]) +
                       (int64_t)by * (c == 0 ? d.dst_stride[0] : c == 1 ? d.dst_stride[1] : d.dst_stride[2]) +
                       (int64_t)bx * E;
        if (E == 64) {                            // dense blocks: 128 B, 16-B aligned
#pragma unroll
          for (int w = 0; w < 8; ++w) reinterpret_cast<uint4*>(out)[w] = reinterpret_cast<const uint4*>(blk)[w];
        } else if (E == 1) {
          *out = blk[0];
        } else {
          for (int w = 0; w < E / 4; ++w)         // E*2 bytes (a multiple of 8): 8-byte words
            reinterpret_cast<uint2*>(out)[w] = reinterpret_cast<const uint2*>(blk)[w];
        }
      }
      if (E == 64) {
#pragma unroll
        for (int w = 0; w < 8; ++w) reinterpret_cast<uint4*>(blk)[w] = make_uint4(0u, 0u, 0u, 0u);
      } else {
        for (int w = 0; w < (E + 3) / 4; ++w) reinterpret_cast<uint2*>(blk)[w] = make_uint2(0u, 0u);
      }
    }
    k = 0;
    if (++x == H) {
      x = 0;
      if (++y == V) {
        y = 0;
        if (++c == nc) {
          c = 0;
          if (++m > m1) break;
          if (++mx == d.mcus_x) { mx = 0; ++my; }
        }
        H = nc == 1 ? 1 : (c == 0 ? d.h[0] : 1);
        V = nc == 1 ? 1 : (c == 0 ? d.v[0] : 1);
        const int td = c == 0 ? d.td[0] : c == 1 ? d.td[1] : d.td[2];
        const int ta = c == 0 ? d.ta[0] : c == 1 ? d.ta[1] : d.ta[2];
        tdc = &d.tabs->dc[td];
        tac = &d.tabs->ac[ta];
        sdc = one_set && td < 2 ? td : -1;
        sac = one_set && ta < 2 ? 2 + ta : -1;
      }
    }
  }
}
#endif

}  // namespace smol
