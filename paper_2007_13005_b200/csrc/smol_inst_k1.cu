// smol_inst_k1.cu -- instantiations of the fused kernel at decode scale
// 1/1 (smol_kernels.cuh); one translation unit per scale so the library
// builds in parallel.
#include "smol_kernels.cuh"
#include "smol_launch.h"

namespace smol {
namespace {

template <int NT> struct CfgYP {
  static constexpr int yp = NT == kThreadsNarrow ? kYPNarrow : NT == kThreadsTiny ? kYPTiny : kYPWide;
};

template <bool PK, int NT, bool DB = false, bool GC = false, int CK = 1>
KernelFn pick(bool f16, bool dbg) {
  constexpr int YP = CfgYP<NT>::yp;
  if (dbg) return f16 ? smol_fused_kernel<1, true, true, PK, NT, YP, DB, GC, CK> : smol_fused_kernel<1, false, true, PK, NT, YP, DB, GC, CK>;
  return f16 ? smol_fused_kernel<1, true, false, PK, NT, YP, DB, GC, CK> : smol_fused_kernel<1, false, false, PK, NT, YP, DB, GC, CK>;
}

template <int NT>
KernelFn pick_nt(bool f16, bool dbg, bool packed, bool db) {
  (void)db;                     // Definitions A and B coincide at this scale
  (void)packed;                 // scale 1: the packed layout is DENSE64
  return pick<false, NT>(f16, dbg);
}

}  // namespace

KernelFn select_fused_k1(bool f16, bool dbg, bool packed, int nt, bool db, bool gc, bool c2s) {
  (void)c2s;                    // (no chroma at twice the scale at scale 1)
  if (gc) return pick<false, kThreadsWide, false, true>(f16, dbg);
  return nt == kThreadsNarrow ? pick_nt<kThreadsNarrow>(f16, dbg, packed, db)
       : nt == kThreadsTiny   ? pick_nt<kThreadsTiny>(f16, dbg, packed, db)
                              : pick_nt<kThreadsWide>(f16, dbg, packed, db);
}

cudaError_t upload_basis_k1(const Basis& b) { return cudaMemcpyToSymbol(c_basis, &b, sizeof(Basis)); }

}  // namespace smol
