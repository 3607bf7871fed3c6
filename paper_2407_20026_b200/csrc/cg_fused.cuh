// Grid barrier and beta epilogue shared by the fused CG update kernels
// (cg_update_fused_kernel in pcg.cu, cg_update_block_fused_kernel in block_jacobi.cu).
//
// A fused update forms r^T z and r^T r over the grid (last-CTA reduction), the last
// CTA writes beta / the convergence test into the state and advances st->gen; every
// other CTA waits for the generation to move, then all form p_next = z + beta p.
// All CTAs are co-resident by construction (grid bounded by the occupancy, launched
// on an otherwise idle stream after the SpMV); the wait is still bounded so that a
// broken launch reports SSO_E_CUDA instead of hanging the device.
#pragma once

#include "sso_internal.h"

namespace sso {

__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Thread 0 of each CTA.  last: this CTA did the final reduction (v = r^T z, r^T r).
// Returns 1 when the CTA may proceed to the p update.
__device__ __forceinline__ int cg_fused_epilogue(bool last, const double (&v)[2], CgState* st, unsigned gen0) {
  if (last) {
    const double rz_new = v[0];
    st->beta = rz_new / st->rz;
    st->rz_prev = st->rz;
    st->rz = rz_new;
    st->rr = v[1];
    st->iter += 1;
    st->pfix = 0;
    if (v[1] <= st->tol2) {
      st->done = 1;
      st->status = SSO_OK;
    } else if (st->iter >= st->max_iter) {
      st->done = 1;
      st->status = SSO_E_NOT_CONVERGED;
    }
    __threadfence();
    atomicAdd(&st->gen, 1u);  // release the grid
    return 1;
  }
  for (int spin = 0; spin < (1 << 22); ++spin) {  // ~0.3 s at most
    if (ld_acquire_u32(&st->gen) != gen0) return 1;
    __nanosleep(64);
  }
  st->status = SSO_E_CUDA;
  st->done = 1;
  return 0;
}

}  // namespace sso
