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
// Decoding per symbol: a 9-bit lookup (length, symbol) for short codes, the
// T.81 F.16 MAXCODE walk for longer ones; bit buffer of 64 bits refilled a
// byte at a time with 0xFF00 unstuffing (B.1.1.5); at a marker the reader
// feeds zero bits (well-formed data never needs them).
#pragma once
#include <stdint.h>

#include "smol_geom.cuh"

namespace smol {

constexpr int kHuffLutBits = 9;

// One Huffman table in the decoder's format (built on the host from a DHT).
struct HuffTable {
  uint16_t lut[1 << kHuffLutBits];   // code prefix -> length << 8 | symbol (length 0: longer code)
  int32_t maxcode[18];               // per length l: largest code of length l (-1: none); [17] sentinel
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
constexpr int kJpegThreads = 128;
constexpr int kJpegBlkStride = 68;   // int16 per thread block buffer (136 B: spreads the lanes' banks)

// warp per image: segment s > 0 starts after the s-th RST marker.  The
// warp reads 512 B per step (16-byte loads, files 16-B aligned), four steps
// in flight; a marker's second byte may sit in the next lane's (or step's)
// first byte.
constexpr int kIndexUnroll = 4;
__global__ void __launch_bounds__(128) smol_jpeg_index_kernel(const JpegDesc* ds, int n_images,
                                                              int32_t* seg_start, int32_t* seg_img) {
  const int lane = threadIdx.x & 31;
  const int img = blockIdx.x * 4 + (threadIdx.x >> 5);
  if (img >= n_images) return;
  const JpegDesc& d = ds[img];
  const uint8_t* p = d.data;
  const int end = d.size, s0 = d.scan_off;
  const int base = d.seg_base, nseg = d.nseg;
  for (int s = lane; s < nseg; s += 32) {         // defaults: segment 0 at the scan start,
    seg_img[base + s] = img;                      // missing markers -> empty segments
    seg_start[base + s] = s == 0 ? s0 : end;
  }
  __syncwarp();
  if (nseg <= 1) return;
  int found = 0;                                  // markers seen so far (whole warp)
  const int a0 = s0 & ~15;
  for (int o = a0; o < end && found < nseg - 1; o += 512 * kIndexUnroll) {
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
      // bit j: 0xFF at byte j and 0xD0..0xD7 at byte j + 1, at or after the scan start
      const uint32_t wd[5] = {w[u].x, w[u].y, w[u].z, w[u].w, nxt};
      uint32_t hits = 0;
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const uint32_t b0 = (wd[j >> 2] >> (8 * (j & 3))) & 0xFFu;
        const uint32_t b1 = j == 15 ? nxt : (wd[(j + 1) >> 2] >> (8 * ((j + 1) & 3))) & 0xFFu;
        if (b0 == 0xFFu && (b1 & 0xF8u) == 0xD0u && q + j >= s0 && q + j + 1 < end) hits |= 1u << j;
      }
      const int cnt = __popc(hits);
      int inc = cnt;                              // inclusive warp scan of the counts
#pragma unroll
      for (int k = 1; k < 32; k <<= 1) {
        const int t = __shfl_up_sync(0xffffffffu, inc, k);
        if (lane >= k) inc += t;
      }
      int idx = found + inc - cnt;                // markers before this lane's first hit
      while (hits) {
        const int j = __ffs(hits) - 1;
        hits &= hits - 1;
        ++idx;                                    // the idx-th marker starts segment idx
        if (idx < nseg) seg_start[base + idx] = q + j + 2;
      }
      found += __shfl_sync(0xffffffffu, inc, 31);
    }
  }
}

struct BitReader {
  const uint8_t* p;
  const uint8_t* pend;
  uint64_t buf;              // left-aligned: next bit is bit 63
  int nb;                    // valid bits in buf
  bool stop;                 // met a marker / the end: feed zeros

  __device__ __forceinline__ void refill() {
    while (nb <= 56) {
      uint32_t b = 0;
      if (!stop) {
        if (p < pend) {
          b = __ldg(p);
          ++p;
          if (b == 0xFFu) {
            const uint32_t b2 = p < pend ? __ldg(p) : 0xD9u;
            if (b2 == 0u) ++p;                    // stuffed 0xFF00 (B.1.1.5)
            else { stop = true; b = 0; }          // a marker ends the interval
          }
        } else {
          stop = true;
        }
      }
      buf |= (uint64_t)b << (56 - nb);
      nb += 8;
    }
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

// T.81 F.16 DECODE (needs >= 16 valid bits)
__device__ __forceinline__ int huff_decode(BitReader& br, const HuffTable* t) {
  const uint32_t look = br.peek16();
  const uint32_t e = __ldg(&t->lut[look >> (16 - kHuffLutBits)]);
  if (e >> 8) {
    br.skip((int)(e >> 8));
    return (int)(e & 255u);
  }
  int l = kHuffLutBits + 1;
  while (l <= 16 && (int32_t)(look >> (16 - l)) > __ldg(&t->maxcode[l])) ++l;
  if (l > 16) { br.skip(16); return 0; }        // invalid code: read as EOB / zero
  br.skip(l);
  return (int)__ldg(&t->huffval[((int32_t)(look >> (16 - l)) + __ldg(&t->valoff[l])) & 255]);
}

// thread per restart interval
__global__ void __launch_bounds__(kJpegThreads) smol_jpeg_decode_kernel(const JpegDesc* ds, int nseg_total,
                                                                        const int32_t* seg_start,
                                                                        const int32_t* seg_img,
                                                                        const int8_t* dst_index) {
  __shared__ __align__(16) int16_t blkbuf[kJpegThreads * kJpegBlkStride];
  __shared__ uint8_t zmap[64];                    // zig-zag position -> stored element (255: dropped)
  if (threadIdx.x < 64) zmap[threadIdx.x] = (uint8_t)dst_index[threadIdx.x];
  int16_t* blk = blkbuf + threadIdx.x * kJpegBlkStride;
#pragma unroll
  for (int i = 0; i < 16; ++i) reinterpret_cast<uint2*>(blk)[i] = make_uint2(0u, 0u);   // (8-B aligned buffers)
  __syncthreads();
  const int g = blockIdx.x * kJpegThreads + threadIdx.x;
  if (g >= nseg_total) return;
  const JpegDesc& d = ds[seg_img[g]];
  const int s = g - d.seg_base;
  const int m0 = s * d.ri, m1 = min(d.nmcu, m0 + d.ri) - 1;
  const int nc = d.ncomp;
  // skip an interval none of whose blocks is inside the ROI box
  {
    const int my0 = m0 / d.mcus_x, my1 = m1 / d.mcus_x;
    const int mxa = my0 == my1 ? m0 - my0 * d.mcus_x : 0;
    const int mxb = my0 == my1 ? m1 - my1 * d.mcus_x : d.mcus_x - 1;
    bool any = false;
    for (int c = 0; c < nc; ++c) {
      const int H = nc == 1 ? 1 : d.h[c], V = nc == 1 ? 1 : d.v[c];
      const int r0 = my0 * V, r1 = my1 * V + V - 1, c0 = mxa * H, c1 = mxb * H + H - 1;
      any |= r0 <= d.by0[c] + d.nby[c] - 1 && r1 >= d.by0[c] && c0 <= d.bx0[c] + d.nbx[c] - 1 && c1 >= d.bx0[c];
    }
    if (!any || m1 < m0) return;
  }
  BitReader br;
  br.p = d.data + seg_start[g];
  br.pend = d.data + d.size;
  br.buf = 0;
  br.nb = 0;
  br.stop = false;
  const int E = d.E;
  int32_t pred0 = 0, pred1 = 0, pred2 = 0;        // DC predictors (reset per interval, F.2.1.3.1)
  for (int m = m0; m <= m1; ++m) {
    const int my = m / d.mcus_x, mx = m - my * d.mcus_x;
    for (int c = 0; c < nc; ++c) {
      const int H = nc == 1 ? 1 : d.h[c], V = nc == 1 ? 1 : d.v[c];
      const HuffTable* tdc = &d.tabs->dc[d.td[c]];
      const HuffTable* tac = &d.tabs->ac[d.ta[c]];
      for (int y = 0; y < V; ++y)
        for (int x = 0; x < H; ++x) {
          // DC (F.2.2.1)
          br.refill();
          const int t = huff_decode(br, tdc);
          const int32_t diff = br.receive_extend(t & 15);
          int32_t& pred = c == 0 ? pred0 : c == 1 ? pred1 : pred2;
          pred += diff;
          const int by = my * V + y - d.by0[c], bx = mx * H + x - d.bx0[c];
          const bool keep = by >= 0 && by < d.nby[c] && bx >= 0 && bx < d.nbx[c];
          blk[0] = (int16_t)pred;                 // zig-zag 0 is stored element 0 in every layout
          // AC (F.2.2.2, Figure F.13)
          for (int k = 1; k < 64;) {
            br.refill();
            const int rs = huff_decode(br, tac);
            const int ssss = rs & 15, r = rs >> 4;
            if (ssss == 0) {
              if (r != 15) break;                 // EOB
              k += 16;                            // ZRL
              continue;
            }
            k += r;
            if (k > 63) break;                    // corrupt run: stop the block
            const int32_t v = br.receive_extend(ssss);
            const int e = zmap[k];
            if (e != 255) blk[e] = (int16_t)v;
            ++k;
          }
          if (keep) {
            int16_t* out = (c == 0 ? d.dst[0] : c == 1 ? d.dst[1] : d.dst[2]) +
                           (int64_t)by * (c == 0 ? d.dst_stride[0] : c == 1 ? d.dst_stride[1] : d.dst_stride[2]) +
                           (int64_t)bx * E;
            if (E == 1) {
              *out = blk[0];
            } else {
              // E*2 bytes (a multiple of 8): 8-byte words
              for (int w = 0; w < E / 4; ++w)
                reinterpret_cast<uint2*>(out)[w] = reinterpret_cast<const uint2*>(blk)[w];
            }
          }
          for (int w = 0; w < (E + 3) / 4; ++w) reinterpret_cast<uint2*>(blk)[w] = make_uint2(0u, 0u);
        }
    }
  }
}
#endif

}  // namespace smol
