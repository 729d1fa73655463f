// smol_compact.cuh -- compact coefficient transport (include/smol_preproc.h
// "Compact coefficient transport"): record format constants,
// the per-scale element-use mask, and the device kernel that expands records
// back into ROI block rows of the plan's layout.
#pragma once
#include <stdint.h>

#include "smol_geom.cuh"

namespace smol {

constexpr uint32_t kCompactMagic = 0x32434D53u;   // "SMC2"
constexpr int kCompactHeader = 64;

struct CompactHeader {            // the 64-byte record header
  uint32_t magic, E, n_units, zero;      // n_units: u16 units of the entry stream
  int32_t bx0[3], by0[3], nbx[3], nby[3];
};
static_assert(sizeof(CompactHeader) == kCompactHeader, "compact header is 64 bytes");

// Bit e set <=> element e of a stored block (layout DENSE64 or PACKED at
// scale 1/K) enters the decode at that scale (Definition B: u, v < 8/K;
// Definition A, reading R1: the box-averaged
// basis of frequency u vanishes exactly for u = 4 at K = 2, u in {2, 4, 6} at
// K = 4, u > 0 at K = 8).  PACKED blocks store exactly the used set (49 / 25
// / 1 elements) followed by zero padding.
inline uint64_t used_mask(int K, bool packed, bool db = false) {
  if (K == 1) return ~0ull;
  if (db) {                       // Definition B (R16): the top-left N x N, N = 8/K
    const int N = 8 / K;
    if (packed) return N * N >= 64 ? ~0ull : (1ull << (N * N)) - 1;
    uint64_t m = 0;
    for (int v = 0; v < N; ++v)
      for (int u = 0; u < N; ++u) m |= 1ull << (v * 8 + u);
    return m;
  }
  if (packed) return K == 2 ? (1ull << 49) - 1 : K == 4 ? (1ull << 25) - 1 : 1ull;
  auto keep = [K](int f) {
    return K == 2 ? f != 4 : K == 4 ? (f == 0 || (f & 1)) : f == 0;
  };
  uint64_t m = 0;
  for (int v = 0; v < 8; ++v)
    for (int u = 0; u < 8; ++u)
      if (keep(u) && keep(v)) m |= 1ull << (v * 8 + u);
  return m;
}

// Entry of one nonzero coefficient: u16 = pos | v << 6 (pos = element index
// in the stored block, v = value as 10-bit two's complement) for
// -511 <= v <= 511; otherwise the escape pos | (-512 << 6) followed by the
// int16 value in the next unit.
constexpr int kEscape = -512;

// Record section offsets (bytes) for `nblocks` ROI blocks in `nrows` block
// rows: u8 block lengths (units) at 64, u32 row starts (4-B aligned), entry
// stream (16-B aligned; at least 2 zero bytes follow it, so a 32-bit load of
// the last unit stays inside the record).
SMOL_HD int64_t compact_rowstart_off(int64_t nblocks) { return (kCompactHeader + nblocks + 3) & ~3LL; }
SMOL_HD int64_t compact_entries_off(int64_t nblocks, int64_t nrows) {
  return (compact_rowstart_off(nblocks) + 4 * nrows + 15) & ~15LL;
}
SMOL_HD int64_t compact_record_bytes(int64_t nblocks, int64_t nrows, int64_t nunits) {
  return (compact_entries_off(nblocks, nrows) + 2 * nunits + 2 + 15) & ~15LL;
}

// One image to expand: record (device) -> staged ROI rows of the plan's layout.
struct ExpandDesc {
  const uint8_t* rec;        // device copy of the record
  int16_t* dst[3];           // staged element (row by0, element bx0 * E) per component
  int32_t dst_stride[3];     // int16 elements per staged row
  int32_t nbx[3], nby[3];    // ROI blocks per row / block rows
  int32_t E;                 // elements per block
};

#if defined(__CUDACC__)
constexpr int kExpandWarps = 4;
// per-lane block buffers are padded by 8 bytes (lane stride 2E + 8 bytes) so
// the lanes' zeroing/scatter stores do not all land in one shared-memory bank
constexpr int kExpandLanePad = 8;               // int16 elements (lane stride 2E + 16 B: 16-B aligned)
constexpr int kExpandBlkBuf = 32 * (64 + kExpandLanePad);
// dynamic shared memory per CTA: per warp a 32-block output buffer
constexpr int kExpandSmem = kExpandWarps * kExpandBlkBuf * 2;
constexpr int kExpandSplit = 8;                 // CTAs per image (block rows interleaved)

// kExpandSplit CTAs per image (block rows interleaved); a warp expands one ROI
// block row at a time, 32 blocks (one per lane) per chunk:
//   1. each lane reads its block's entry length; a warp scan gives each
//      block's first entry;
//   2. each lane reads its block's entries straight from the record (the
//      chunk's entries are contiguous, so neighbouring lanes share L1 lines);
//   3. each lane zeroes its block in a shared buffer and scatters its entries
//      into it;
//   4. the chunk's 32 blocks are contiguous in the staged row: the warp copies
//      the buffer out with coalesced 8-byte stores.
// E = 1 (DC plane): lane per block, direct store.
__global__ void __launch_bounds__(kExpandWarps * 32) smol_expand_kernel(const ExpandDesc* eds) {
  extern __shared__ __align__(16) uint8_t esm[];
  const ExpandDesc e = eds[blockIdx.x / kExpandSplit];
  const int part = blockIdx.x % kExpandSplit;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int16_t* blk = reinterpret_cast<int16_t*>(esm) + warp * kExpandBlkBuf;
  const int E = e.E;
  const uint32_t fd_wpb = make_fastdiv((uint32_t)(E / 4 > 0 ? E / 4 : 1)).m;
  // component bases without dynamically indexed arrays (no local memory)
  const int nb0 = e.nbx[0] * e.nby[0], nb1 = e.nbx[1] * e.nby[1], nb2 = e.nbx[2] * e.nby[2];
  const int r1 = e.nby[0], r2 = e.nby[0] + e.nby[1], nrows = r2 + e.nby[2];
  const int nblocks = nb0 + nb1 + nb2;
  const uint8_t* len_all = e.rec + kCompactHeader;
  const uint32_t* rowst = reinterpret_cast<const uint32_t*>(e.rec + compact_rowstart_off(nblocks));
  const uint16_t* units = reinterpret_cast<const uint16_t*>(e.rec + compact_entries_off(nblocks, nrows));
  // record-supplied counts are clamped (a corrupt record must not make this
  // kernel read or write out of bounds): units per block <= 2 E (<= 128),
  // every staged unit inside the record's n_units
  const uint32_t n_units = reinterpret_cast<const CompactHeader*>(e.rec)->n_units;
  const int max_len = 2 * E < 128 ? 2 * E : 128;
  for (int gr = part * kExpandWarps + warp; gr < nrows; gr += kExpandWarps * kExpandSplit) {
    const int c = gr >= r2 ? 2 : gr >= r1 ? 1 : 0;
    const int r = gr - (c == 2 ? r2 : c == 1 ? r1 : 0);
    const int nbx = c == 2 ? e.nbx[2] : c == 1 ? e.nbx[1] : e.nbx[0];
    const uint8_t* lens = len_all + (c == 2 ? nb0 + nb1 : c == 1 ? nb0 : 0) + (int64_t)r * nbx;
    int16_t* const dst_c = c == 2 ? e.dst[2] : c == 1 ? e.dst[1] : e.dst[0];
    const int stride_c = c == 2 ? e.dst_stride[2] : c == 1 ? e.dst_stride[1] : e.dst_stride[0];
    int16_t* drow = dst_c + (int64_t)r * stride_c;
    uint32_t vbase = min(__ldg(rowst + gr), n_units);
    for (int ch = 0; ch < nbx; ch += 32) {
      const int b = ch + lane;
      const int cnt = b < nbx ? min((int)__ldg(lens + b), max_len) : 0;   // units of this block's entries
      int inc = cnt;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += t;
      }
      // this lane's units are [inc - cnt, inc) of the chunk; a row overrunning
      // the record is cut at n_units (later blocks' ranges shrink to nothing)
      const int total = min(__shfl_sync(0xffffffffu, inc, 31), (int)(n_units - vbase));
      const int first = min(inc - cnt, total);
      const int cntc = min(inc, total) - first;
      // 2. each lane reads its own entries straight from the record (the
      // chunk's units are contiguous: neighbouring lanes share L1 lines), so
      // no shared staging -- 3x more resident warps to hide the load latency
      const uint16_t* ub = units + vbase + first;
      const int nb = min(32, nbx - ch);
      if (E == 1) {
        __syncwarp();
        if (b < nbx) {
          int16_t v = 0;
          if (cntc) {
            v = (int16_t)__ldg(ub) >> 6;
            if (v == kEscape) v = (int16_t)__ldg(ub + 1);
          }
          drow[b] = v;
        }
      } else {
        // 3. zero + scatter this lane's block (E*2 bytes, a multiple of 8)
        const int ls = E + kExpandLanePad;                 // lane stride (elements)
        int16_t* mine = blk + lane * ls;
        if (E % 8 == 0) {                                   // (dense: 16-byte words)
          uint4* m16 = reinterpret_cast<uint4*>(mine);
          for (int q = 0; q < E / 8; ++q) m16[q] = make_uint4(0u, 0u, 0u, 0u);
        } else {
          uint2* m8 = reinterpret_cast<uint2*>(mine);
          for (int q = 0; q < E / 4; ++q) m8[q] = make_uint2(0u, 0u);
        }
        __syncwarp();                                       // staged entries visible
        for (int j = 0; j < cntc; ++j) {
          const uint16_t u = __ldg(ub + j);
          int16_t v = (int16_t)u >> 6;
          if (v == kEscape) v = (int16_t)__ldg(ub + (++j));
          mine[u & 63] = v;
        }
        __syncwarp();
        // 4. copy the nb blocks out (contiguous in the staged row): word w of
        // the chunk is word w % wpb of block w / wpb; 16-byte words when the
        // blocks are (dense: 128 B blocks, 16-B aligned rows), else 8-byte
        if (E % 8 == 0) {
          const int wpb = E / 8;                            // 16-byte words per block
          uint4* to16 = reinterpret_cast<uint4*>(drow + (int64_t)ch * E);
          for (int w = lane; w < nb * wpb; w += 32) {
            const int bb = w / wpb;
            to16[w] = reinterpret_cast<const uint4*>(blk + bb * ls)[w - bb * wpb];
          }
        } else {
          const int wpb = E / 4;                            // 8-byte words per block
          uint2* to8 = reinterpret_cast<uint2*>(drow + (int64_t)ch * E);
          for (int w = lane; w < nb * wpb; w += 32) {
            const int bb = wpb == 1 ? w : (int)__umulhi((uint32_t)w, fd_wpb);   // w / wpb (w < 2^16)
            to8[w] = reinterpret_cast<const uint2*>(blk + bb * ls)[w - bb * wpb];
          }
        }
      }
      __syncwarp();
      vbase += (uint32_t)total;
    }
  }
}
#endif

}  // namespace smol
