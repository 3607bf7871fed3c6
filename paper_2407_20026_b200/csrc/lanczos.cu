// A3 certification — extreme Ritz values of the preconditioned operator from the CG
// coefficients, and the end-of-solve sums for the error estimates (sm_100a).
//
// PAPER.md:71-74 (Eq. 1) is solved by CG (north star); SURVEY §8(c) C5 asks for the
// Lanczos extreme Ritz values formed from (alpha, beta) to bound the error.  CG with
// x0 = 0 is the Lanczos process on M^-1 K; its tridiagonal T_m (m iterations) has
//     T[k][k]   = 1 / alpha_k + beta_{k-1} / alpha_{k-1}     (beta_{-1} = 0)
//     T[k][k+1] = sqrt(beta_k) / alpha_k
// (oracle: oracle/solve.py lanczos_ritz, which forms T and calls eigvalsh).  Here:
//   lanczos_tridiag_kernel  (d_k, e_k^2) of T for every recorded iteration, in parallel;
//   lanczos_ritz_kernel     one CTA per (design, extreme): Gershgorin interval, then
//                           multisection with 128 shifts per round on the Sturm count of
//                           T - s I, evaluated by the three-term recurrence of the leading
//                           principal minors (one FMA per step on the dependency chain, exact
//                           power-of-two rescaling, no division) over shared-memory tiles of T.  lambda_max on
//                           a linear grid, lambda_min on a geometric grid (T is SPD: its
//                           smallest eigenvalue can sit many decades below the largest);
//                           rounds stop at 1e-10 relative width.
//   cert_sums_kernel        at the converged x: |r|^2, r^T M^-1 r, f^T x, x^T x with the TRUE
//                           residual r = f_bc - K x (thread per node, point or block M).
// Ritz values lie inside the spectrum (interlacing), so lambda_min(T) >= lambda_min(M^-1 K):
// the error figures built from it in api.cu are estimates, exact once T has resolved the
// smallest eigenvalue (which CG does by convergence).
#include <cfloat>
#include <cmath>

#include "cg_common.cuh"
#include "sso_internal.h"

namespace sso {

namespace {

constexpr int RITZ_THREADS = 128;  // the recurrence is issue-bound: few warps, more rounds

__global__ void __launch_bounds__(256) lanczos_tridiag_kernel(const CgState* st, double2* T, int cap) {
  const int bd = blockIdx.y;
  const CgState* S = st + bd;
  T += (int64_t)bd * cap;
  const int n = S->lz_n;
  const double* h = S->lz;
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) {
    const double a = h[2 * k];
    double d = 1.0 / a;
    if (k > 0) d += h[2 * (k - 1) + 1] / h[2 * (k - 1)];
    const double e2 = (k + 1 < n) ? h[2 * k + 1] / (a * a) : 0.0;
    T[k] = make_double2(d, e2);
  }
}

// Sturm count state of one shift: the number of eigenvalues of T below s = sign changes of the
// leading principal minors p_0 = 1, p_1 = d_0 - s, p_{k+1} = (d_k - s) p_k - e_{k-1}^2 p_{k-1}
// (negative LDL^T pivots).  Advanced over a shared-memory tile of T (every thread of the CTA
// walks the same entries: broadcast reads), four steps between exact power-of-two rescalings
// (the pair's magnitude changes by far less than 2^500 in four steps): the dependency chain is
// one FMA per step.
struct Sturm {
  double pp, p, e2;
  int cnt;
  __device__ void start(double2 t0, double s) {
    pp = 1.0;
    p = t0.x - s;
    cnt = p < 0.0;
    e2 = t0.y;
  }
  __device__ __forceinline__ void step(double2 t, double s) {
    const double pn = fma(t.x - s, p, -e2 * pp);
    cnt += ((pn < 0.0) != (p < 0.0)) || pn == 0.0;
    pp = p;
    p = pn;
    e2 = t.y;
  }
  __device__ __forceinline__ void rescale() {
    const double m = fmax(fabs(p), fabs(pp));
    if (m > 0x1p+500) {
      p *= 0x1p-500;
      pp *= 0x1p-500;
    } else if (m < 0x1p-500 && m > 0.0) {
      p *= 0x1p+500;
      pp *= 0x1p+500;
    }
  }
  // entries [k0, k1) of the tile (k0 >= 1 globally handled by the caller)
  __device__ void run(const double2* tile, int k0, int k1, double s) {
    int k = k0;
    for (; k + 3 < k1; k += 4) {
      const double2 t0 = tile[k], t1 = tile[k + 1], t2 = tile[k + 2], t3 = tile[k + 3];
      step(t0, s);
      step(t1, s);
      step(t2, s);
      step(t3, s);
      rescale();
    }
    for (; k < k1; ++k) step(tile[k], s);
    rescale();
  }
};

constexpr int RITZ_TILE = 2048;  // double2 entries of T per shared-memory tile (32 KB)

// count(s) for this thread's shift over all n entries of T, tile by tile (all threads call it)
__device__ int sturm_count_tiled(const double2* __restrict__ T, int n, double s, double2* tile) {
  Sturm S;
  for (int base = 0; base < n; base += RITZ_TILE) {
    const int len = min(RITZ_TILE, n - base);
    __syncthreads();
    for (int i = threadIdx.x; i < len; i += blockDim.x) tile[i] = T[base + i];
    __syncthreads();
    if (base == 0) {
      S.start(tile[0], s);
      S.run(tile, 1, len, s);
    } else {
      S.run(tile, 0, len, s);
    }
  }
  return S.cnt;
}

__global__ void __launch_bounds__(RITZ_THREADS) lanczos_ritz_kernel(CgState* st, const double2* T, int cap) {
  const int bd = blockIdx.y, which = blockIdx.x;  // 0: lambda_min, 1: lambda_max
  CgState* S = st + bd;
  T += (int64_t)bd * cap;
  const int n = S->lz_n;
  __shared__ double s_lo[RITZ_THREADS], s_hi[RITZ_THREADS];
  __shared__ int s_cnt[RITZ_THREADS];
  __shared__ double2 tile[RITZ_TILE];
  __shared__ double s_a, s_b;
  if (n <= 0) {
    if (threadIdx.x == 0) {
      if (which == 0) S->lz_min = nan("");
      else S->lz_max = nan("");
    }
    return;
  }
  // Gershgorin interval
  double lo = DBL_MAX, hi = -DBL_MAX;
  for (int k = threadIdx.x; k < n; k += blockDim.x) {
    const double r = (k > 0 ? sqrt(T[k - 1].y) : 0.0) + sqrt(T[k].y);
    lo = fmin(lo, T[k].x - r);
    hi = fmax(hi, T[k].x + r);
  }
  s_lo[threadIdx.x] = lo;
  s_hi[threadIdx.x] = hi;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int i = 1; i < RITZ_THREADS; ++i) {
      lo = fmin(lo, s_lo[i]);
      hi = fmax(hi, s_hi[i]);
    }
    hi = hi + 1e-12 * fabs(hi) + DBL_MIN;
    if (which == 1) {
      s_a = lo;
      s_b = hi;
    } else {
      s_a = (lo > 0.0) ? lo : hi * 0x1p-110;  // T is SPD in exact arithmetic
      s_b = hi;
    }
  }
  __syncthreads();
  for (int round = 0; round < 12; ++round) {
    const double a = s_a, b = s_b;
    if (which == 1 ? (b - a) <= 1e-10 * fabs(b) : (b / a - 1.0) <= 1e-10) break;
    const double f = (double)(threadIdx.x + 1) / (RITZ_THREADS + 1);
    const double s = which == 1 ? a + (b - a) * f : a * exp2(log2(b / a) * f);
    s_lo[threadIdx.x] = s;
    s_cnt[threadIdx.x] = sturm_count_tiled(T, n, s, tile);
    __syncthreads();
    if (threadIdx.x == 0) {
      if (which == 1) {  // first shift with all n eigenvalues below it
        int t = 0;
        while (t < RITZ_THREADS && s_cnt[t] < n) ++t;
        s_a = t > 0 ? s_lo[t - 1] : a;
        s_b = t < RITZ_THREADS ? s_lo[t] : b;
      } else {  // first shift with an eigenvalue below it
        int t = 0;
        while (t < RITZ_THREADS && s_cnt[t] < 1) ++t;
        s_a = t > 0 ? s_lo[t - 1] : a;
        s_b = t < RITZ_THREADS ? s_lo[t] : b;
      }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    const double v = 0.5 * (s_a + s_b);
    if (which == 0) S->lz_min = v;
    else S->lz_max = v;
  }
}

// |r|^2, r^T M^-1 r, f^T x, x^T x at the converged x (r = f_bc - K x, Kx given); point
// Jacobi (dinv) or node-block Jacobi (binv); thread per node; red[0..3] via the last CTA.
__global__ void __launch_bounds__(256) cert_sums_kernel(int n_nodes, const double* __restrict__ fbc,
                                                        const double* __restrict__ Kx,
                                                        const double* __restrict__ x,
                                                        const double* __restrict__ dinv,
                                                        const double* __restrict__ binv, double* partial,
                                                        CgState* st, BatchStrides bs) {
  __shared__ double sm[32 * 4];
  {
    const int bd = blockIdx.y;
    fbc += bd * bs.dof;
    Kx += bd * bs.dof;
    x += bd * bs.dof;
    if (dinv) dinv += bd * bs.dof;
    if (binv) binv += (int64_t)bd * 21 * n_nodes;
    partial += bd * bs.partial;
    st += bd;
  }
  double v[4] = {0.0, 0.0, 0.0, 0.0};
  for (int64_t n = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; n < n_nodes;
       n += (int64_t)gridDim.x * blockDim.x) {
    double f6[6], k6[6], x6[6], r[6], z[6];
    ld6(fbc, n, f6);
    ld6(Kx, n, k6);
    ld6(x, n, x6);
#pragma unroll
    for (int a = 0; a < 6; ++a) r[a] = f6[a] - k6[a];
    if (binv) {
      block_apply(binv, n_nodes, n, r, z);
    } else {
      double d6[6];
      ld6(dinv, n, d6);
#pragma unroll
      for (int a = 0; a < 6; ++a) z[a] = d6[a] * r[a];
    }
#pragma unroll
    for (int a = 0; a < 6; ++a) {
      v[0] += r[a] * r[a];
      v[1] += r[a] * z[a];
      v[2] += f6[a] * x6[a];
      v[3] += x6[a] * x6[a];
    }
  }
  if (grid_sum<4>(v, partial, &st->ticket[3], sm) && threadIdx.x == 0) {
#pragma unroll
    for (int k = 0; k < 4; ++k) st->red[k] = v[k];
  }
}

// Scale of M for the 2-norm estimate: min over DOFs of 1/dinv (point) or over nodes of
// 1/|(K_nn)^-1|_F <= lambda_min(K_nn) (block); positive doubles compare as their bit
// patterns, so an atomicMin on them is exact and order-independent.
__global__ void __launch_bounds__(256) mscale_kernel(int n_nodes, const double* __restrict__ dinv,
                                                     const double* __restrict__ binv,
                                                     unsigned long long* out, BatchStrides bs) {
  const int bd = blockIdx.y;
  if (dinv) dinv += bd * bs.dof;
  if (binv) binv += (int64_t)bd * 21 * n_nodes;
  double m = DBL_MAX;
  for (int64_t n = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; n < n_nodes;
       n += (int64_t)gridDim.x * blockDim.x) {
    if (binv) {
      double f2 = 0.0;
#pragma unroll
      for (int a = 0; a < 6; ++a)
#pragma unroll
        for (int b = a; b < 6; ++b) {
          const double w = binv[(int64_t)tri6(a, b) * n_nodes + n];
          f2 += (a == b ? 1.0 : 2.0) * w * w;
        }
      m = fmin(m, 1.0 / sqrt(f2));
    } else {
#pragma unroll
      for (int a = 0; a < 6; ++a) m = fmin(m, 1.0 / dinv[6 * n + a]);
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = fmin(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0 && m > 0.0) atomicMin(out + bd, (unsigned long long)__double_as_longlong(m));
}

}  // namespace

void launch_lanczos_ritz(cudaStream_t s, CgState* st, double* Tbuf, int cap, int B) {
  if (cap <= 0) return;
  double2* T = reinterpret_cast<double2*>(Tbuf);
  const int g = std::min((cap + 255) / 256, cg_grid());
  lanczos_tridiag_kernel<<<dim3(g, B), 256, 0, s>>>(st, T, cap);
  SSO_POST_LAUNCH("lanczos_tridiag_kernel");
  lanczos_ritz_kernel<<<dim3(2, B), RITZ_THREADS, 0, s>>>(st, T, cap);
  SSO_POST_LAUNCH("lanczos_ritz_kernel");
}

void launch_cert_sums(cudaStream_t s, int n_nodes, const double* fbc, const double* Kx, const double* x,
                      const double* dinv, const double* binv, double* partial, CgState* st, const BatchStrides& bs) {
  const int g = std::max(1, std::min((n_nodes + 255) / 256, cg_grid() / bs.B));
  cert_sums_kernel<<<dim3(g, bs.B), 256, 0, s>>>(n_nodes, fbc, Kx, x, binv ? nullptr : dinv, binv, partial, st, bs);
  SSO_POST_LAUNCH("cert_sums_kernel");
}

void launch_mscale(cudaStream_t s, int n_nodes, const double* dinv, const double* binv, unsigned long long* out,
                   const BatchStrides& bs) {
  const int g = std::max(1, std::min((n_nodes + 255) / 256, cg_grid() / bs.B));
  mscale_kernel<<<dim3(g, bs.B), 256, 0, s>>>(n_nodes, binv ? nullptr : dinv, binv, out, bs);
  SSO_POST_LAUNCH("mscale_kernel");
}

}  // namespace sso
