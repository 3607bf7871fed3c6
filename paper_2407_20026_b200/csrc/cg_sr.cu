// A3 on partitioned handles — single-reduction Jacobi-PCG (sm_100a).
//
// The PCG of reading c10 (Eq. 1; x0 = 0, M = diag(K_bc) or the node blocks,
// stop |r| <= rtol |f_bc|) rearranged after Chronopoulos & Gear so that every iteration needs
// ONE global reduction instead of two: with u = M^-1 r, w = K u, s = K p,
//     gamma_i = r_i^T u_i,  delta_i = u_i^T w_i,  beta_i = gamma_i / gamma_{i-1},
//     alpha_i = gamma_i / (delta_i - beta_i gamma_i / alpha_{i-1})     (= gamma_i / p_i^T K p_i)
//     p = u + beta p,  s = w + beta s,  x += alpha p,  r -= alpha s,  u = M^-1 r
// (exact-arithmetic identical iterates to the textbook loop of oracle/solve.py pcg; the first
// iteration and every restart take beta = 0, alpha = gamma / delta).  Per iteration:
//     halo of u -> SpMV w = K u with the local delta (red[0]) -> allreduce of red[0..3]
//     (delta, gamma, r^T r, |f_bc|^2 on the first pass) -> update (red[1], red[2] local).
// No scalar kernels: every CTA of the update forms alpha, beta and the convergence test from
// the allreduced values (identical in every CTA and on every rank); the last CTA records the
// state.  The convergence test sees r^T r of the residual the previous update formed, so a
// solve performs one SpMV more than it has iterations.  Lanczos pairs (alpha_{i-1}, beta_i)
// are recorded at iteration i (lanczos.cu).  Vector traffic: 96 B per DOF per iteration
// (u, w, p, s, x, r, M read; p, s, x, r, u written).
#include "cg_common.cuh"
#include "sso_internal.h"

namespace sso {

namespace {

__device__ __forceinline__ void apply_M(const double* __restrict__ dinv, const double* __restrict__ binv, int64_t nn,
                                        int64_t n, const double (&r)[6], double (&u)[6]) {
  if (binv) {
    block_apply(binv, nn, n, r, u);
  } else {
    double d[6];
    ld6(dinv, n, d);
#pragma unroll
    for (int a = 0; a < 6; ++a) u[a] = d[a] * r[a];
  }
}

__global__ void __launch_bounds__(256) cgsr_init_kernel(int n_own, const double* __restrict__ f,
                                                        const uint8_t* __restrict__ fixed_mask,
                                                        const double* __restrict__ dinv,
                                                        const double* __restrict__ binv, double* __restrict__ fbc,
                                                        double* __restrict__ x, double* __restrict__ r,
                                                        double* __restrict__ u, double* __restrict__ p,
                                                        double* __restrict__ sv, double* partial, CgState* st,
                                                        int warm, const double* __restrict__ Kx0) {
  __shared__ double sm[32 * 3];
  double v[3] = {0.0, 0.0, 0.0};  // gamma, r^T r, f^T f
  const double zero6[6] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
  for (int64_t n = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; n < n_own; n += (int64_t)gridDim.x * blockDim.x) {
    const unsigned mask = fixed_mask[n];
    double f6[6], r6[6], u6[6];
    ld6(f, n, f6);
#pragma unroll
    for (int a = 0; a < 6; ++a) f6[a] = ((mask >> a) & 1) ? 0.0 : f6[a];
    st6(fbc, n, f6);
    if (warm) {
      double k6[6];
      ld6(Kx0, n, k6);
#pragma unroll
      for (int a = 0; a < 6; ++a) r6[a] = f6[a] - k6[a];
    } else {
#pragma unroll
      for (int a = 0; a < 6; ++a) r6[a] = f6[a];
      st6(x, n, zero6);
    }
    apply_M(dinv, binv, n_own, n, r6, u6);
    st6(r, n, r6);
    st6(u, n, u6);
    st6(p, n, zero6);
    st6(sv, n, zero6);
#pragma unroll
    for (int a = 0; a < 6; ++a) {
      v[0] += r6[a] * u6[a];
      v[1] += r6[a] * r6[a];
      v[2] += f6[a] * f6[a];
    }
  }
  if (grid_sum<3>(v, partial, &st->ticket[2], sm) && threadIdx.x == 0) {
    st->red[1] = v[0];
    st->red[2] = v[1];
    st->red[3] = v[2];
  }
}

__global__ void __launch_bounds__(256) cgsr_update_kernel(int n_own, const double* __restrict__ dinv,
                                                          const double* __restrict__ binv, double* __restrict__ x,
                                                          double* __restrict__ r, double* __restrict__ u,
                                                          const double* __restrict__ w, double* __restrict__ p,
                                                          double* __restrict__ sv, double* partial, CgState* st,
                                                          const SrPart* __restrict__ mp) {
  __shared__ double sm[64];
  if (mp) {  // part blockIdx.y of a multi-part launch
    const SrPart& A = mp[blockIdx.y];
    n_own = A.n_own;
    dinv = A.dinv;
    binv = A.binv;
    x = A.x;
    r = A.r;
    u = A.u;
    w = A.w;
    p = A.p;
    sv = A.sv;
    partial = A.partial;
    st = A.st;
  }
  if (st->done) return;
  // allreduced: delta (this iteration's SpMV), gamma and r^T r (the previous update), |f|^2
  const double delta = st->red[0], gamma = st->red[1], rr = st->red[2];
  const double ff = st->ff < 0.0 ? st->red[3] : st->ff;
  const double tol = st->tol2_rel * ff;
  const long long it = st->iter;
  const bool first = it == 0 || st->sr_restart;
  const double alpha_prev = st->alpha;
  double beta = 0.0, den = delta;
  if (!first) {
    beta = gamma / st->rz;
    den = delta - beta * gamma / alpha_prev;  // = p^T K p of the new p
  }
  const bool conv = rr <= tol || ff == 0.0;
  const bool maxed = it >= st->max_iter;
  const bool bad = !(den > 0.0);
  if (conv || maxed || bad) {
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      st->ff = ff;
      st->tol2 = tol;
      st->rr = rr;
      st->pq = den;
      st->status = conv ? SSO_OK : (bad ? SSO_E_NOT_SPD : SSO_E_NOT_CONVERGED);
      if (!first) lz_record(st, alpha_prev, 0.0);  // the last alpha (its beta is never formed)
      st->done = 1;
    }
    return;
  }
  const double alpha = gamma / den;
  double v[2] = {0.0, 0.0};
  for (int64_t n = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; n < n_own; n += (int64_t)gridDim.x * blockDim.x) {
    double u6[6], w6[6], p6[6], s6[6], x6[6], r6[6];
    ld6(u, n, u6);
    ld6(w, n, w6);
    ld6(p, n, p6);
    ld6(sv, n, s6);
    ld6(x, n, x6);
    ld6(r, n, r6);
#pragma unroll
    for (int a = 0; a < 6; ++a) {
      p6[a] = fma(beta, p6[a], u6[a]);
      s6[a] = fma(beta, s6[a], w6[a]);
      x6[a] = fma(alpha, p6[a], x6[a]);
      r6[a] = fma(-alpha, s6[a], r6[a]);
    }
    apply_M(dinv, binv, n_own, n, r6, u6);
    st6(p, n, p6);
    st6(sv, n, s6);
    st6(x, n, x6);
    st6(r, n, r6);
    st6(u, n, u6);
#pragma unroll
    for (int a = 0; a < 6; ++a) {
      v[0] += r6[a] * u6[a];
      v[1] += r6[a] * r6[a];
    }
  }
  if (grid_sum<2>(v, partial, &st->ticket[1], sm) && threadIdx.x == 0) {
    if (!first) lz_record(st, alpha_prev, beta);
    st->red[1] = v[0];
    st->red[2] = v[1];
    st->red[3] = 0.0;  // |f|^2 travels once
    st->ff = ff;
    st->tol2 = tol;
    st->alpha = alpha;
    st->beta = beta;
    st->rz = gamma;
    st->rr = rr;
    st->pq = den;
    st->iter = it + 1;
    st->sr_restart = 0;
  }
}

// Restart at the true residual for the designs cg_check selected (reliable >= 1): r = f_bc - K x,
// u = M^-1 r, local gamma and r^T r into red[1], red[2]; the next iteration takes beta = 0.
__global__ void __launch_bounds__(256) cgsr_replace_kernel(int n_own, const double* __restrict__ fbc,
                                                           const double* __restrict__ Kx,
                                                           const double* __restrict__ dinv,
                                                           const double* __restrict__ binv, double* __restrict__ r,
                                                           double* __restrict__ u, double* partial, CgState* st) {
  __shared__ double sm[64];
  if (!st->act) return;
  double v[2] = {0.0, 0.0};
  for (int64_t n = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; n < n_own; n += (int64_t)gridDim.x * blockDim.x) {
    double f6[6], k6[6], r6[6], u6[6];
    ld6(fbc, n, f6);
    ld6(Kx, n, k6);
#pragma unroll
    for (int a = 0; a < 6; ++a) r6[a] = f6[a] - k6[a];
    apply_M(dinv, binv, n_own, n, r6, u6);
    st6(r, n, r6);
    st6(u, n, u6);
#pragma unroll
    for (int a = 0; a < 6; ++a) {
      v[0] += r6[a] * u6[a];
      v[1] += r6[a] * r6[a];
    }
  }
  if (grid_sum<2>(v, partial, &st->ticket[1], sm) && threadIdx.x == 0) {
    st->red[1] = v[0];
    st->red[2] = v[1];
    st->red[3] = 0.0;
    st->rr_ref = v[1];
    st->sr_restart = 1;
    st->act = 0;
  }
}

__global__ void __launch_bounds__(256) halo_gather_kernel(int n_ent, const int4* __restrict__ ent,
                                                          double* const* __restrict__ base) {
  const int64_t n = 6 * (int64_t)n_ent;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int4 e = ent[i / 6];
    const int c = (int)(i % 6);
    base[e.x][6 * (int64_t)e.y + c] = base[e.z][6 * (int64_t)e.w + c];
  }
}

int vgrid(int64_t n) { return (int)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, cg_grid())); }

}  // namespace

void launch_cgsr_init(cudaStream_t s, int n_own, const double* f, const uint8_t* fixed_mask, const double* dinv,
                      const double* binv, double* fbc, double* x, double* r, double* u, double* p, double* sv,
                      double* partial, CgState* st, int warm, const double* Kx0) {
  cgsr_init_kernel<<<vgrid(n_own), 256, 0, s>>>(n_own, f, fixed_mask, binv ? nullptr : dinv, binv, fbc, x, r, u, p,
                                                sv, partial, st, warm, Kx0);
  SSO_POST_LAUNCH("cgsr_init_kernel");
}

void launch_cgsr_update(cudaStream_t s, int n_own, const double* dinv, const double* binv, double* x, double* r,
                        double* u, const double* w, double* p, double* sv, double* partial, CgState* st, int share) {
  const int g = std::max(1, vgrid(n_own) / std::max(share, 1));
  cgsr_update_kernel<<<g, 256, 0, s>>>(n_own, binv ? nullptr : dinv, binv, x, r, u, w, p, sv, partial, st, nullptr);
  SSO_POST_LAUNCH("cgsr_update_kernel");
}

void launch_cgsr_update_multi(cudaStream_t s, const SrPart* mp, int n_parts, int max_own) {
  if (n_parts <= 0) return;
  const int g = std::max(1, vgrid(max_own) / n_parts);
  cgsr_update_kernel<<<dim3(g, n_parts), 256, 0, s>>>(max_own, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr,
                                                      nullptr, nullptr, nullptr, nullptr, mp);
  SSO_POST_LAUNCH("cgsr_update_kernel (parts)");
}

void launch_cgsr_replace(cudaStream_t s, int n_own, const double* fbc, const double* Kx, const double* dinv,
                         const double* binv, double* r, double* u, double* partial, CgState* st) {
  cgsr_replace_kernel<<<vgrid(n_own), 256, 0, s>>>(n_own, fbc, Kx, binv ? nullptr : dinv, binv, r, u, partial, st);
  SSO_POST_LAUNCH("cgsr_replace_kernel");
}

void launch_halo_gather(cudaStream_t s, int n_ent, const int4* ent, double* const* base) {
  if (n_ent <= 0) return;
  halo_gather_kernel<<<vgrid(6 * (int64_t)n_ent), 256, 0, s>>>(n_ent, ent, base);
  SSO_POST_LAUNCH("halo_gather_kernel");
}

}  // namespace sso
