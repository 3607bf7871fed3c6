// Grid all-reduce shared by the fused CG update kernels (cg_update_fused_kernel in pcg.cu,
// cg_update_block_fused_kernel in block_jacobi.cu).
//
// A fused update forms r^T z and r^T r over the grid: every CTA publishes its two partials,
// counts itself in (one atomic), waits until all CTAs of its design have arrived, then sums
// ALL partials itself in one fixed order -- every CTA obtains bit-identical totals, forms beta
// and the convergence test locally and goes on to p_next = z + beta p with no second
// release step; CTA 0 records the state.  All CTAs are co-resident: the grid is bounded by
// the occupancy and the kernels are launched cooperatively (launch_cooperative in
// sso_internal.h: the driver co-schedules the whole grid or rejects the launch).  The wait is
// still bounded (2^23 polls with a 20 ns back-off: a few seconds at most) so that a broken
// launch reports SSO_E_CUDA instead of hanging the device.
#pragma once

#include "sso_internal.h"

namespace sso {

__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ double fused_warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// v: this thread's (r^T z, r^T r) partials in, the grid totals out (every thread).  part:
// 2 doubles per CTA; arrive: the design's monotonic arrival counter (+gridDim.x per launch).
// sm: 64 doubles of shared memory.  Returns 0 if the arrival wait timed out.
__device__ __forceinline__ int cg_fused_allreduce(double (&v)[2], double* part, unsigned* arrive, double* sm) {
  __shared__ int s_ok;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const unsigned G = gridDim.x;
  double a0 = fused_warp_sum(v[0]), a1 = fused_warp_sum(v[1]);
  if (lane == 0) {
    sm[2 * w] = a0;
    sm[2 * w + 1] = a1;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double c0 = 0.0, c1 = 0.0;
    for (int i = 0; i < nw; ++i) {
      c0 += sm[2 * i];
      c1 += sm[2 * i + 1];
    }
    part[2 * blockIdx.x] = c0;
    part[2 * blockIdx.x + 1] = c1;
    __threadfence();
    const unsigned old = atomicAdd(arrive, 1u);
    const unsigned target = (old / G + 1) * G;
    int ok = 0;
    for (int spin = 0; spin < (1 << 23); ++spin) {  // a few seconds at most
      if ((int)(ld_acquire_u32(arrive) - target) >= 0) {
        ok = 1;
        break;
      }
      __nanosleep(20);
    }
    s_ok = ok;
  }
  __syncthreads();
  if (!s_ok) return 0;
  a0 = a1 = 0.0;
  for (unsigned b = threadIdx.x; b < G; b += blockDim.x) {
    a0 += __ldcg(part + 2 * b);
    a1 += __ldcg(part + 2 * b + 1);
  }
  a0 = fused_warp_sum(a0);
  a1 = fused_warp_sum(a1);
  if (lane == 0) {
    sm[2 * w + 32] = a0;  // second half: the first half may still be read above
    sm[2 * w + 33] = a1;
  }
  __syncthreads();
  double t0 = 0.0, t1 = 0.0;
  for (int i = 0; i < nw; ++i) {  // every thread, the same order
    t0 += sm[2 * i + 32];
    t1 += sm[2 * i + 33];
  }
  v[0] = t0;
  v[1] = t1;
  return 1;
}

// alpha = r^T z / p^T q at the start of a fused update.  With st->defer_alpha the SpMV left
// st->npq partials of p^T q at pq_part: every CTA sums them in one fixed order (bit-identical
// in all CTAs); otherwise the SpMV's last CTA already stored alpha.  Returns 0 (all CTAs) when
// p^T q <= 0: CTA 0 records SSO_E_NOT_SPD.
__device__ __forceinline__ int cg_fused_alpha(const double* pq_part, CgState* st, double* sm, double rz_old,
                                             double& alpha, double& pqv) {
  if (!st->defer_alpha) {
    alpha = st->alpha;
    pqv = st->pq;
    return 1;
  }
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int np = st->npq;
  double a = 0.0;
  for (int b = threadIdx.x; b < np; b += blockDim.x) a += __ldcg(pq_part + b);
  a = fused_warp_sum(a);
  if (lane == 0) sm[w] = a;
  __syncthreads();
  double t = 0.0;
  for (int i = 0; i < nw; ++i) t += sm[i];  // every thread, the same order
  __syncthreads();                          // sm is reused by the all-reduce
  pqv = t;
  if (!(t > 0.0)) {
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      st->pq = t;
      st->status = SSO_E_NOT_SPD;
      st->done = 1;
    }
    return 0;
  }
  alpha = rz_old / t;
  return 1;
}

// beta and the convergence test from the grid totals; CTA 0 records the state.  Returns 1
// when the caller goes on to the p update (not converged / not stopped).
__device__ __forceinline__ int cg_fused_step(const double (&v)[2], CgState* st, double rz_old, long long iter_old,
                                            double alpha, double pqv, double& beta) {
  const double rz_new = v[0], rr = v[1];
  beta = rz_new / rz_old;
  const bool conv = rr <= st->tol2;
  const bool maxed = iter_old + 1 >= st->max_iter;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    st->alpha = alpha;
    st->pq = pqv;
    st->beta = beta;
    st->rz_prev = rz_old;
    st->rz = rz_new;
    st->rr = rr;
    st->iter = iter_old + 1;
    st->pfix = 0;
    lz_record(st, alpha, beta);
    if (conv) {
      st->done = 1;
      st->status = SSO_OK;
    } else if (maxed) {
      st->done = 1;
      st->status = SSO_E_NOT_CONVERGED;
    }
  }
  return !(conv || maxed);
}

}  // namespace sso
