// Device helpers shared by the CG kernels (pcg.cu, block_jacobi.cu, lanczos.cu):
// fixed-order block / grid sums (per-CTA partials, last-CTA reduction: bit-reproducible
// for a fixed grid), 6-vector loads / stores and the packed node-block apply of the
// node-block Jacobi preconditioner.
#pragma once

#include "sso_internal.h"

namespace sso {

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Block-wide sum of NV values (fixed order); result valid in thread 0.
template <int NV>
__device__ __forceinline__ void block_sum(double (&v)[NV], double* sm /*[32*NV]*/) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
  for (int k = 0; k < NV; ++k) v[k] = warp_sum(v[k]);
  if (lane == 0)
#pragma unroll
    for (int k = 0; k < NV; ++k) sm[w * NV + k] = v[k];
  __syncthreads();
  if (w == 0) {
#pragma unroll
    for (int k = 0; k < NV; ++k) {
      double s = (lane < nw) ? sm[lane * NV + k] : 0.0;
      v[k] = warp_sum(s);
    }
  }
  __syncthreads();
}

// Write this CTA's partials; returns true in the last CTA to arrive, which then
// owns the fixed-order final reduction (result in thread 0 of that CTA).
template <int NV>
__device__ __forceinline__ bool grid_sum(double (&v)[NV], double* partial, unsigned int* ticket,
                                         double* sm) {
  __shared__ bool last;
  block_sum<NV>(v, sm);
  if (threadIdx.x == 0) {
#pragma unroll
    for (int k = 0; k < NV; ++k) partial[(int64_t)blockIdx.x * NV + k] = v[k];
    __threadfence();
    unsigned int t = atomicAdd(ticket, 1u);
    last = (t == gridDim.x - 1);
  }
  __syncthreads();
  if (!last) return false;
  __threadfence();
  double acc[NV];
#pragma unroll
  for (int k = 0; k < NV; ++k) acc[k] = 0.0;
  for (int b = threadIdx.x; b < (int)gridDim.x; b += blockDim.x)
#pragma unroll
    for (int k = 0; k < NV; ++k) acc[k] += __ldcg(partial + (int64_t)b * NV + k);
  block_sum<NV>(acc, sm);
#pragma unroll
  for (int k = 0; k < NV; ++k) v[k] = acc[k];
  if (threadIdx.x == 0) *ticket = 0u;  // re-arm for the next launch
  return true;
}

// Node-block Jacobi (precond 1): the packed upper triangle of (K_nn)^-1, row-major:
// entry (a, b), a <= b, at a*6 - a(a-1)/2 + b-a.
__device__ __forceinline__ int tri6(int a, int b) { return a * 6 - (a * (a - 1)) / 2 + (b - a); }

// 6-vector loads / stores at 6 n (48-byte aligned)
__device__ __forceinline__ void ld6(const double* __restrict__ v, int64_t n, double (&o)[6]) {
  const double2* p = reinterpret_cast<const double2*>(v + 6 * n);
  const double2 a = p[0], b = p[1], c = p[2];
  o[0] = a.x; o[1] = a.y; o[2] = b.x; o[3] = b.y; o[4] = c.x; o[5] = c.y;
}
__device__ __forceinline__ void st6(double* __restrict__ v, int64_t n, const double (&o)[6]) {
  double2* p = reinterpret_cast<double2*>(v + 6 * n);
  p[0] = make_double2(o[0], o[1]);
  p[1] = make_double2(o[2], o[3]);
  p[2] = make_double2(o[4], o[5]);
}

// z = Binv_n r (packed symmetric), fixed-order sums
__device__ __forceinline__ void block_apply(const double* __restrict__ binv, int64_t nn, int64_t n,
                                            const double (&r)[6], double (&z)[6]) {
  double m[21];
#pragma unroll
  for (int e = 0; e < 21; ++e) m[e] = binv[e * nn + n];
#pragma unroll
  for (int a = 0; a < 6; ++a) {
    double s = 0.0;
#pragma unroll
    for (int b = 0; b < 6; ++b) s = fma(m[a <= b ? tri6(a, b) : tri6(b, a)], r[b], s);
    z[a] = s;
  }
}


}  // namespace sso
