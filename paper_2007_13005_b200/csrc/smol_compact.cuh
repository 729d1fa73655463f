// smol_compact.cuh -- compact coefficient transport (include/smol_preproc.h
// "Compact coefficient transport"): record format constants,
// the per-scale element-use mask, and the device kernel that expands records
// back into ROI block rows of the plan's layout.
#pragma once
#include <stdint.h>

#include "smol_geom.cuh"

namespace smol {

constexpr uint32_t kCompactMagic = 0x31434D53u;   // "SMC1"
constexpr int kCompactHeader = 64;

struct CompactHeader {            // the 64-byte record header
  uint32_t magic, E, n_values, zero;
  int32_t bx0[3], by0[3], nbx[3], nby[3];
};
static_assert(sizeof(CompactHeader) == kCompactHeader, "compact header is 64 bytes");

// Bit e set <=> element e of a stored block (layout DENSE64 or PACKED at
// scale 1/K) enters the decode at that scale (reading R1: the box-averaged
// basis of frequency u vanishes exactly for u = 4 at K = 2, u in {2, 4, 6} at
// K = 4, u > 0 at K = 8).  PACKED blocks store exactly the used set (49 / 25
// / 1 elements) followed by zero padding.
inline uint64_t used_mask(int K, bool packed) {
  if (K == 1) return ~0ull;
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

// Record section offsets (bytes) for `nblocks` ROI blocks in `nrows` block rows.
SMOL_HD int64_t compact_rowstart_off(int64_t nblocks) { return kCompactHeader + 8 * nblocks; }
SMOL_HD int64_t compact_values_off(int64_t nblocks, int64_t nrows) {
  return (compact_rowstart_off(nblocks) + 4 * nrows + 15) & ~15LL;
}
// (at least 2 zero bytes follow the values, so a 32-bit load of the last value
// stays inside the record)
SMOL_HD int64_t compact_record_bytes(int64_t nblocks, int64_t nrows, int64_t nvalues) {
  return (compact_values_off(nblocks, nrows) + 2 * nvalues + 2 + 15) & ~15LL;
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
constexpr int kExpandWarps = 8;
constexpr int kExpandChunkVals = 32 * 64 + 8;  // values of one 32-block chunk (worst case) + alignment slack

// One CTA per image; a warp expands one ROI block row at a time, 32 blocks
// per chunk: each lane reads one bitmap, a warp scan of the popcounts gives
// each block's first value; the chunk's values (contiguous in the record) are
// copied to the warp's shared-memory buffer with independent coalesced loads
// (so the dependent per-block gathers below hit shared memory, not HBM
// latency); then the warp writes the chunk's blocks one after another: lane
// l produces elements 2l, 2l+1 (one coalesced 32-bit store per lane, a 128-B
// block per warp instruction at E = 64).  E = 1 (DC plane): lane per block.
__global__ void __launch_bounds__(kExpandWarps * 32) smol_expand_kernel(const ExpandDesc* eds) {
  __shared__ int16_t sv[kExpandWarps][kExpandChunkVals];
  const ExpandDesc e = eds[blockIdx.x];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int16_t* buf = sv[warp];
  int blk_base[3], row_base[3];
  int nblocks = 0, nrows = 0;
  for (int c = 0; c < 3; ++c) {
    blk_base[c] = nblocks; row_base[c] = nrows;
    nblocks += e.nbx[c] * e.nby[c];
    nrows += e.nby[c];
  }
  const uint64_t* bm_all = reinterpret_cast<const uint64_t*>(e.rec + kCompactHeader);
  const uint32_t* rowst = reinterpret_cast<const uint32_t*>(e.rec + compact_rowstart_off(nblocks));
  const int16_t* vals = reinterpret_cast<const int16_t*>(e.rec + compact_values_off(nblocks, nrows));
  for (int gr = warp; gr < nrows; gr += kExpandWarps) {
    const int c = gr >= row_base[2] ? 2 : gr >= row_base[1] ? 1 : 0;
    const int r = gr - row_base[c];
    const int nbx = e.nbx[c];
    const uint64_t* bm = bm_all + blk_base[c] + (int64_t)r * nbx;
    int16_t* drow = e.dst[c] + (int64_t)r * e.dst_stride[c];
    uint32_t vbase = __ldg(rowst + gr);
    for (int ch = 0; ch < nbx; ch += 32) {
      const int b = ch + lane;
      const uint64_t m = b < nbx ? __ldg(bm + b) : 0ull;
      const int cnt = __popcll(m);
      int inc = cnt;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += t;
      }
      const int first = inc - cnt;                       // relative to the chunk
      const int total = __shfl_sync(0xffffffffu, inc, 31);
      // stage the chunk's values: 32-bit loads from the 4-B aligned start
      const int16_t* src = vals + vbase;
      const int mis = (int)(reinterpret_cast<uintptr_t>(src) & 3) >> 1;     // 0 or 1 element
      const uint32_t* s32 = reinterpret_cast<const uint32_t*>(src - mis);
      const int nw = (total + mis + 1) >> 1;
      uint32_t* b32 = reinterpret_cast<uint32_t*>(buf);
      for (int w = lane; w < nw; w += 32) b32[w] = __ldg(s32 + w);
      __syncwarp();
      const int16_t* cv = buf + mis;
      const int nb = min(32, nbx - ch);
      if (e.E == 1) {
        if (b < nbx) drow[b] = m ? cv[first] : (int16_t)0;
      } else {
        const int e0 = 2 * lane;
        for (int j = 0; j < nb; ++j) {
          const uint64_t mj = __shfl_sync(0xffffffffu, m, j);
          const int fj = __shfl_sync(0xffffffffu, first, j);
          if (e0 < e.E) {
            const int k = fj + __popcll(mj & ((1ull << e0) - 1ull));
            const uint32_t b0 = (uint32_t)(mj >> e0) & 1u, b1 = (uint32_t)(mj >> (e0 + 1)) & 1u;
            const uint32_t v0 = b0 ? (uint16_t)cv[k] : 0u;
            const uint32_t v1 = b1 ? (uint16_t)cv[k + b0] : 0u;
            *reinterpret_cast<uint32_t*>(drow + (int64_t)(ch + j) * e.E + e0) = v0 | (v1 << 16);
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
