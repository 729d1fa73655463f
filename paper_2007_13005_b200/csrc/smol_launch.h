// smol_launch.h -- kernel instantiation units of the fused kernel (one per
// decode scale, compiled in parallel: smol_inst_k{1,2,4,8}.cu) and the host
// runtime (smol_preproc.cu) meet here.
#pragma once
#include <cuda_runtime.h>

namespace smol {

struct KParams;
struct Basis;
using KernelFn = void (*)(const KParams);

// fused kernel instantiation for (scale 1/K, output dtype, debug store,
// packed layout, threads per CTA, Definition B IDCT); K fixed per unit
// (db only exists at K = 2, 4: at 1 and 1/8 the definitions coincide);
// gc: generic-chroma kernel (4:2:2 / 4:4:4), built for the wide CTA only
// (nt is ignored); c2s (with gc, K >= 2, dense, Definition A): chroma blocks
// decoded at scale 1/(K/2) (reading R18)
KernelFn select_fused_k1(bool f16, bool dbg, bool packed, int nt, bool db, bool gc, bool c2s);
KernelFn select_fused_k2(bool f16, bool dbg, bool packed, int nt, bool db, bool gc, bool c2s);
KernelFn select_fused_k4(bool f16, bool dbg, bool packed, int nt, bool db, bool gc, bool c2s);
KernelFn select_fused_k8(bool f16, bool dbg, bool packed, int nt, bool db, bool gc, bool c2s);
// upload the basis constants into each unit's constant bank (current device)
cudaError_t upload_basis_k1(const Basis& b);
cudaError_t upload_basis_k2(const Basis& b);
cudaError_t upload_basis_k4(const Basis& b);
cudaError_t upload_basis_k8(const Basis& b);

}  // namespace smol
