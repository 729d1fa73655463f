// smol_inst_k4.cu -- instantiations of the fused kernel at decode scale
// 1/4 (smol_kernels.cuh); one translation unit per scale so the library
// builds in parallel.
#include "smol_kernels.cuh"
#include "smol_launch.h"

namespace smol {
namespace {

template <int NT> struct CfgYP {
  static constexpr int yp = NT == kThreadsNarrow ? kYPNarrow : NT == kThreadsTiny ? kYPTiny : kYPWide;
};

template <bool PK, int NT, bool DB = false, bool GC = false, int CK = 4>
KernelFn pick(bool f16, bool dbg) {
  constexpr int YP = CfgYP<NT>::yp;
  if (dbg) return f16 ? smol_fused_kernel<4, true, true, PK, NT, YP, DB, GC, CK> : smol_fused_kernel<4, false, true, PK, NT, YP, DB, GC, CK>;
  return f16 ? smol_fused_kernel<4, true, false, PK, NT, YP, DB, GC, CK> : smol_fused_kernel<4, false, false, PK, NT, YP, DB, GC, CK>;
}

template <int NT>
KernelFn pick_nt(bool f16, bool dbg, bool packed, bool db) {
  if (db) return packed ? pick<true, NT, true>(f16, dbg) : pick<false, NT, true>(f16, dbg);
  return packed ? pick<true, NT>(f16, dbg) : pick<false, NT>(f16, dbg);
}

}  // namespace

KernelFn select_fused_k4(bool f16, bool dbg, bool packed, int nt, bool db, bool gc, bool c2s) {
  if (c2s) return pick<false, kThreadsWide, false, true, 2>(f16, dbg);   // chroma at 1/2 (R18)
  if (gc) {
    constexpr int W = kThreadsWide;
    if (db) return packed ? pick<true, W, true, true>(f16, dbg) : pick<false, W, true, true>(f16, dbg);
    return packed ? pick<true, W, false, true>(f16, dbg) : pick<false, W, false, true>(f16, dbg);
  }
  return nt == kThreadsNarrow ? pick_nt<kThreadsNarrow>(f16, dbg, packed, db)
       : nt == kThreadsTiny   ? pick_nt<kThreadsTiny>(f16, dbg, packed, db)
                              : pick_nt<kThreadsWide>(f16, dbg, packed, db);
}

cudaError_t upload_basis_k4(const Basis& b) { return cudaMemcpyToSymbol(c_basis, &b, sizeof(Basis)); }

}  // namespace smol
