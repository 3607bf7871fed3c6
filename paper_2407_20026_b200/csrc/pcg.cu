// A3 — fp64 Jacobi-preconditioned CG kernels (sm_100a), SURVEY.md §8(a) A3.
//
// Solves K_bc u = f_bc (Eq. 1; supports by elimination, reading
// c1) with the CG of reading c10: x0 = 0, M = diag(K_bc), stop when
// |r|_2 <= rtol |f_bc|_2, breakdown p^T K p <= 0 -> NOT_SPD.
//
// One iteration = 3 kernels, all HBM-bound, no host synchronisation:
//   spmv_dot  q = K p and p^T q; the last CTA forms alpha = r^T z / p^T q
//   update    x += alpha p, r -= alpha q, z = dinv r; partial r^T z, r^T r;
//             the last CTA forms beta, tests convergence, sets `done`
//   pupdate   p = dinv r + beta p
// Every kernel returns immediately once `done` is set, so a fixed chunk of
// iterations can be captured once in a CUDA graph and replayed; the host only
// polls `done` between chunks.  Reductions are atomic-free: per-CTA partials
// in fixed order, reduced by the last CTA to finish (ticket counter) in fixed
// order -> bit-reproducible for a fixed grid.
//
// SpMV layout: the scalar CSR values of node n's six rows are contiguous at
// 36 node_ptr[n]; row 6n+a, column 6m+b with m = node_col[node_ptr[n]+k] sits at
// 36 node_ptr[n] + a (6 deg) + 6k + b.  One warp per node: lane rem walks the
// row positions, gathers p[6m+b] ONCE and applies it to all six rows (6
// coalesced value streams); a 9-shuffle transposed butterfly reduces the six
// row sums.  Column indices are read per 6x6 block (4 B / 36 values) instead
// of per value (4 B / value): 8.1 B per non-zero instead of 12.
#include <climits>
#include <cstdio>

#include "sso_internal.h"

namespace sso {

long long g_launches = 0;
static char g_launch_err[256] = {0};
void note_launch_error(const char* name, cudaError_t e) {
  if (!g_launch_err[0]) snprintf(g_launch_err, sizeof g_launch_err, "%s: %s", name, cudaGetErrorString(e));
}
const char* last_launch_error() { return g_launch_err; }

namespace {

int g_sms = 0;

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

// Transposed butterfly: reduce 6 (padded to 8) per-lane values across the warp
// in 9 shuffles.  On return, lane L holds the total of value index
// vi(L) = 4 bit4(L) + 2 bit3(L) + bit2(L) (valid for every L; lanes sharing vi agree).
__device__ __forceinline__ double reduce6(double (&acc)[8], int lane) {
  const bool b4 = lane & 16, b3 = lane & 8, b2 = lane & 4;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    double send = b4 ? acc[k] : acc[k + 4];
    double keep = b4 ? acc[k + 4] : acc[k];
    acc[k] = keep + __shfl_xor_sync(0xffffffffu, send, 16);
  }
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    double send = b3 ? acc[k] : acc[k + 2];
    double keep = b3 ? acc[k + 2] : acc[k];
    acc[k] = keep + __shfl_xor_sync(0xffffffffu, send, 8);
  }
  {
    double send = b2 ? acc[0] : acc[1];
    double keep = b2 ? acc[1] : acc[0];
    acc[0] = keep + __shfl_xor_sync(0xffffffffu, send, 4);
  }
  acc[0] += __shfl_xor_sync(0xffffffffu, acc[0], 2);
  acc[0] += __shfl_xor_sync(0xffffffffu, acc[0], 1);
  return acc[0];
}

// y = K x for node n (warp-cooperative); returns y[6n + vi(lane)] in every lane.
__device__ __forceinline__ double node_row_products(int64_t n, const int64_t* __restrict__ node_ptr,
                                                    const int32_t* __restrict__ node_col,
                                                    const double* __restrict__ vals,
                                                    const double* __restrict__ x, int lane) {
  const int64_t b0 = node_ptr[n];
  const int deg = (int)(node_ptr[n + 1] - b0);
  const int rowlen = 6 * deg;
  const double* base = vals + 36 * b0;
  double acc[8];
#pragma unroll
  for (int a = 0; a < 8; ++a) acc[a] = 0.0;
#pragma unroll 2
  for (int rem = lane; rem < rowlen; rem += 32) {
    const int k = rem / 6;
    const int b = rem - 6 * k;
    const int m = __ldg(node_col + b0 + k);
    const double xv = x[6 * (int64_t)m + b];
#pragma unroll
    for (int a = 0; a < 6; ++a) acc[a] += __ldcs(base + a * rowlen + rem) * xv;
  }
  return reduce6(acc, lane);
}

__global__ void __launch_bounds__(256) spmv_dot_kernel(
    int n_nodes, const int64_t* __restrict__ node_ptr, const int32_t* __restrict__ node_col,
    const double* __restrict__ vals, const double* __restrict__ p, double* __restrict__ q,
    double* __restrict__ partial, CgState* st) {
  __shared__ double sm[32];
  if (st->done) return;
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int vi = ((lane >> 4) & 1) * 4 + ((lane >> 3) & 1) * 2 + ((lane >> 2) & 1);
  const bool writer = ((lane & 3) == 0) && vi < 6;
  double pq[1] = {0.0};
  for (int64_t n = warp; n < n_nodes; n += nwarps) {
    const double y = node_row_products(n, node_ptr, node_col, vals, p, lane);
    if (writer) {
      q[6 * n + vi] = y;
      pq[0] += p[6 * n + vi] * y;
    }
  }
  if (grid_sum<1>(pq, partial, &st->ticket[0], sm) && threadIdx.x == 0) {
    st->pq = pq[0];
    if (!(pq[0] > 0.0)) {
      st->status = SSO_E_NOT_SPD;
      st->done = 1;
    } else {
      st->alpha = st->rz / pq[0];
    }
  }
}

__global__ void __launch_bounds__(256) spmv_kernel(int n_nodes, const int64_t* __restrict__ node_ptr,
                                                   const int32_t* __restrict__ node_col,
                                                   const double* __restrict__ vals,
                                                   const double* __restrict__ x,
                                                   double* __restrict__ y) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int vi = ((lane >> 4) & 1) * 4 + ((lane >> 3) & 1) * 2 + ((lane >> 2) & 1);
  const bool writer = ((lane & 3) == 0) && vi < 6;
  for (int64_t n = warp; n < n_nodes; n += nwarps) {
    const double v = node_row_products(n, node_ptr, node_col, vals, x, lane);
    if (writer) y[6 * n + vi] = v;
  }
}

__global__ void __launch_bounds__(256) cg_update_kernel(int ndof, const double* __restrict__ dinv,
                                                        double* __restrict__ x,
                                                        double* __restrict__ r,
                                                        const double* __restrict__ p,
                                                        const double* __restrict__ q,
                                                        double* __restrict__ partial,
                                                        CgState* st) {
  __shared__ double sm[64];
  if (st->done) return;
  const double alpha = st->alpha;
  double v[2] = {0.0, 0.0};  // r^T z, r^T r
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < ndof; i += stride) {
    const double xi = x[i] + alpha * p[i];
    const double ri = r[i] - alpha * q[i];
    x[i] = xi;
    r[i] = ri;
    const double zi = dinv[i] * ri;
    v[0] += ri * zi;
    v[1] += ri * ri;
  }
  if (grid_sum<2>(v, partial, &st->ticket[1], sm) && threadIdx.x == 0) {
    const double rz_new = v[0];
    st->beta = rz_new / st->rz;
    st->rz = rz_new;
    st->rr = v[1];
    st->iter += 1;
    if (v[1] <= st->tol2) {
      st->done = 1;
      st->status = SSO_OK;
    } else if (st->iter >= st->max_iter) {
      st->done = 1;
      st->status = SSO_E_NOT_CONVERGED;
    }
  }
}

__global__ void __launch_bounds__(256) cg_pupdate_kernel(int ndof, const double* __restrict__ dinv,
                                                         const double* __restrict__ r,
                                                         double* __restrict__ p,
                                                         const CgState* st) {
  if (st->done) return;
  const double beta = st->beta;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < ndof; i += stride)
    p[i] = dinv[i] * r[i] + beta * p[i];
}

// f_bc = f with fixed DOFs zeroed; x = x0 (fixed zeroed) or 0; r = f_bc - K x0; p = z = dinv r.
__global__ void __launch_bounds__(256) cg_init_kernel(int ndof, const double* __restrict__ f,
                                                      const uint8_t* __restrict__ fixed_mask,
                                                      const double* __restrict__ dinv,
                                                      double* __restrict__ fbc,
                                                      double* __restrict__ x,
                                                      double* __restrict__ r,
                                                      double* __restrict__ p,
                                                      double* __restrict__ partial, CgState* st,
                                                      int warm, const double* __restrict__ Kx0) {
  __shared__ double sm[96];
  double v[3] = {0.0, 0.0, 0.0};  // f^T f, r^T z, r^T r
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < ndof; i += stride) {
    const bool fx = (fixed_mask[i / 6] >> (i % 6)) & 1;
    const double fi = fx ? 0.0 : f[i];
    fbc[i] = fi;
    double ri = fi;
    if (warm) {
      ri = fi - Kx0[i];
    } else {
      x[i] = 0.0;
    }
    r[i] = ri;
    const double zi = dinv[i] * ri;
    p[i] = zi;
    v[0] += fi * fi;
    v[1] += ri * zi;
    v[2] += ri * ri;
  }
  if (grid_sum<3>(v, partial, &st->ticket[2], sm) && threadIdx.x == 0) {
    st->ff = v[0];
    st->rz = v[1];
    st->rr = v[2];
    st->iter = 0;
    st->status = SSO_OK;
    st->done = (v[2] <= st->tol2 * v[0] || v[0] == 0.0) ? 1 : 0;
    st->tol2 = st->tol2 * v[0];  // host passes rtol^2 in tol2; becomes rtol^2 |f_bc|^2
    st->alpha = st->beta = 0.0;
  }
}

// zero fixed entries of x (warm start)
__global__ void zero_fixed_kernel(int ndof, const uint8_t* __restrict__ fixed_mask, double* x) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < ndof; i += stride)
    if ((fixed_mask[i / 6] >> (i % 6)) & 1) x[i] = 0.0;
}

__global__ void __launch_bounds__(256) residual_kernel(int ndof, const double* __restrict__ f,
                                                       const double* __restrict__ Kx,
                                                       double* __restrict__ partial,
                                                       unsigned int* ticket, double* out) {
  __shared__ double sm[32];
  double v[1] = {0.0};
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < ndof; i += stride) {
    const double d = f[i] - Kx[i];
    v[0] += d * d;
  }
  if (grid_sum<1>(v, partial, ticket, sm) && threadIdx.x == 0) *out = v[0];
}

__global__ void __launch_bounds__(256) dot_kernel(int n, const double* __restrict__ a,
                                                  const double* __restrict__ b, double scale,
                                                  double* __restrict__ partial, unsigned int* ticket,
                                                  double* out) {
  __shared__ double sm[32];
  double v[1] = {0.0};
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
    v[0] += a[i] * b[i];
  if (grid_sum<1>(v, partial, ticket, sm) && threadIdx.x == 0) *out = scale * v[0];
}

int vec_grid(int64_t n) {
  int64_t need = (n + 255) / 256;
  return (int)std::max<int64_t>(1, std::min<int64_t>(need, (int64_t)cg_grid()));
}

}  // namespace

int cg_grid() {
  if (g_sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_sms, cudaDevAttrMultiProcessorCount, dev);
    if (g_sms <= 0) g_sms = 148;
  }
  return g_sms * 4;  // 4 CTAs x 256 threads per SM, every grid a multiple of the SM count
}

void launch_cg_init(cudaStream_t s, int ndof, const double* f, const uint8_t* fixed_mask,
                    const double* dinv, double* fbc, double* x, double* r, double* p,
                    double* partial, CgState* st, int warm, const double* Kx0) {
  cg_init_kernel<<<vec_grid(ndof), 256, 0, s>>>(ndof, f, fixed_mask, dinv, fbc, x, r, p, partial,
                                                st, warm, Kx0);
  SSO_POST_LAUNCH("cg_init_kernel");
}

void launch_zero_fixed(cudaStream_t s, int ndof, const uint8_t* fixed_mask, double* x) {
  zero_fixed_kernel<<<vec_grid(ndof), 256, 0, s>>>(ndof, fixed_mask, x);
  SSO_POST_LAUNCH("zero_fixed_kernel");
}

void launch_spmv_dot(cudaStream_t s, int n_nodes, const int64_t* node_ptr,
                     const int32_t* node_col, const double* vals, const double* p, double* q,
                     double* partial, CgState* st) {
  int64_t need = ((int64_t)n_nodes + 7) / 8;
  int grid = (int)std::max<int64_t>(1, std::min<int64_t>(need, (int64_t)cg_grid()));
  spmv_dot_kernel<<<grid, 256, 0, s>>>(n_nodes, node_ptr, node_col, vals, p, q, partial, st);
  SSO_POST_LAUNCH("spmv_dot_kernel");
}

void launch_spmv(cudaStream_t s, int n_nodes, const int64_t* node_ptr, const int32_t* node_col,
                 const double* vals, const double* x, double* y) {
  int64_t need = ((int64_t)n_nodes + 7) / 8;
  int grid = (int)std::max<int64_t>(1, std::min<int64_t>(need, (int64_t)cg_grid()));
  spmv_kernel<<<grid, 256, 0, s>>>(n_nodes, node_ptr, node_col, vals, x, y);
  SSO_POST_LAUNCH("spmv_kernel");
}

void launch_cg_update(cudaStream_t s, int ndof, const double* dinv, double* x, double* r,
                      const double* p, const double* q, double* partial, CgState* st) {
  cg_update_kernel<<<vec_grid(ndof), 256, 0, s>>>(ndof, dinv, x, r, p, q, partial, st);
  SSO_POST_LAUNCH("cg_update_kernel");
}

void launch_cg_pupdate(cudaStream_t s, int ndof, const double* dinv, const double* r, double* p,
                       CgState* st) {
  cg_pupdate_kernel<<<vec_grid(ndof), 256, 0, s>>>(ndof, dinv, r, p, st);
  SSO_POST_LAUNCH("cg_pupdate_kernel");
}

void launch_residual_norm(cudaStream_t s, int ndof, const double* f, const double* Kx,
                          double* partial, unsigned int* ticket, double* out) {
  residual_kernel<<<vec_grid(ndof), 256, 0, s>>>(ndof, f, Kx, partial, ticket, out);
  SSO_POST_LAUNCH("residual_kernel");
}

void launch_dot(cudaStream_t s, int n, const double* a, const double* b, double scale,
                double* partial, unsigned int* ticket, double* out) {
  dot_kernel<<<vec_grid(n), 256, 0, s>>>(n, a, b, scale, partial, ticket, out);
  SSO_POST_LAUNCH("dot_kernel");
}

}  // namespace sso
