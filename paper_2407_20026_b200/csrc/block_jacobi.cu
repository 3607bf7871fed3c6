// A3 variant — node-block Jacobi preconditioner for the PCG (sm_100a).
//
// sso_options.precond = 1 (reading c19): M = blockdiag(K_nn), the 6x6
// diagonal block of every node of K_bc, instead of diag(K_bc).  The CG loop is
// the one of pcg.cu (reading c10) with z = M^-1 r; oracle: oracle/solve.py
// pcg_block.  Shell nodes couple translations and rotations inside the node
// block (global frame), so the block version needs fewer iterations (about 30 %
// fewer on the C3 family) for 6x more preconditioner bytes (21 packed values per
// node instead of 6).
//
// Layout: binv [B][21][n_own] (SoA, coalesced per entry), the packed upper
// triangle of (K_nn)^-1, row-major: entry (a, b), a <= b, at a*6 - a(a-1)/2 + b-a.
// z [B][6 n_own] is stored by the update so that the p update reads one vector.
// Kernels are node-granular (a thread per node, its 6-vectors as 3 double2) and
// keep the atomic-free fixed-order reductions of pcg.cu (same epilogues).
#include "cg_common.cuh"
#include "cg_fused.cuh"
#include "sso_internal.h"

namespace sso {

namespace {


// (K_nn)^-1 of every owned node from the assembled values.  Run layout: 0 full storage
// (row-major runs, diagonal block at its rank in the node's column list), 3 upper-block
// records (PULL_BLOCK, rec_off; diagonal first).
__global__ void __launch_bounds__(128) block_inverse_kernel(int n_nodes, const int64_t* __restrict__ node_ptr,
                                                            const int32_t* __restrict__ node_col,
                                                            const double* __restrict__ vals, int layout,
                                                            double* __restrict__ binv, DevFlags* flags,
                                                            BatchStrides bs) {
  const int bd = blockIdx.y;
  vals += bd * bs.nnz;
  binv += (int64_t)bd * 21 * n_nodes;
  flags += bd;
  const int64_t n = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (n >= n_nodes) return;
  const int64_t b0 = node_ptr[n];
  const int deg = (int)(node_ptr[n + 1] - b0);
  int64_t off;
  int rs, cs;
  if (layout == 0) {
    int k = 0;
    while (k < deg && node_col[b0 + k] != n) ++k;
    off = 36 * b0 + 6 * k;
    rs = 6 * deg;
    cs = 1;
  } else {
    off = PULL_BLOCK * b0;
    rs = cs = 0;  // record layout (rec_off)
  }
  // Cholesky K_nn = L L^T (lower, in place), then (K_nn)^-1 = L^-T L^-1
  double L[6][6];
#pragma unroll
  for (int a = 0; a < 6; ++a)
#pragma unroll
    for (int b = 0; b < 6; ++b) L[a][b] = vals[off + (layout == 3 ? rec_off(a, b) : a * rs + b * cs)];
  bool ok = true;
#pragma unroll
  for (int j = 0; j < 6; ++j) {
    double d = L[j][j];
#pragma unroll
    for (int k = 0; k < j; ++k) d -= L[j][k] * L[j][k];
    ok = ok && d > 0.0;
    const double ljj = sqrt(d > 0.0 ? d : 1.0);
    L[j][j] = ljj;
#pragma unroll
    for (int i = j + 1; i < 6; ++i) {
      double s = L[i][j];
#pragma unroll
      for (int k = 0; k < j; ++k) s -= L[i][k] * L[j][k];
      L[i][j] = s / ljj;
    }
  }
  if (!ok) atomicMin(&flags->singular_dof, (int)(6 * n));
  // W = L^-1 (lower triangular)
  double W[6][6];
#pragma unroll
  for (int a = 0; a < 6; ++a)
#pragma unroll
    for (int b = 0; b < 6; ++b) W[a][b] = 0.0;
#pragma unroll
  for (int j = 0; j < 6; ++j) {
    W[j][j] = 1.0 / L[j][j];
#pragma unroll
    for (int i = j + 1; i < 6; ++i) {
      double s = 0.0;
#pragma unroll
      for (int k = j; k < i; ++k) s -= L[i][k] * W[k][j];
      W[i][j] = s / L[i][i];
    }
  }
  // M = W^T W, packed upper triangle
#pragma unroll
  for (int a = 0; a < 6; ++a)
#pragma unroll
    for (int b = a; b < 6; ++b) {
      double s = 0.0;
#pragma unroll
      for (int k = (a > b ? a : b); k < 6; ++k) s += W[k][a] * W[k][b];
      binv[(int64_t)tri6(a, b) * n_nodes + n] = s;
    }
}

// f_bc, x0, r0 = f_bc - K x0, z0 = M^-1 r0, p0 = z0; f^T f, r^T z, r^T r -> state (init epilogue)
__global__ void __launch_bounds__(256) cg_init_block_kernel(int n_nodes, const double* __restrict__ f,
                                                            const uint8_t* __restrict__ fixed_mask,
                                                            const double* __restrict__ binv,
                                                            double* __restrict__ fbc, double* __restrict__ x,
                                                            double* __restrict__ r, double* __restrict__ p,
                                                            double* __restrict__ z, double* __restrict__ partial,
                                                            CgState* st, int warm, const double* __restrict__ Kx0,
                                                            BatchStrides bs) {
  __shared__ double sm[96];
  {
    const int bd = blockIdx.y;
    f += bd * bs.dof;
    binv += (int64_t)bd * 21 * n_nodes;
    fbc += bd * bs.dof;
    x += bd * bs.dof;
    r += bd * bs.dof;
    p += bd * bs.dof;
    z += bd * bs.dof;
    Kx0 += bd * bs.dof;
    partial += bd * bs.partial;
    st += bd;
  }
  double v[3] = {0.0, 0.0, 0.0};
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t n = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; n < n_nodes; n += stride) {
    const unsigned mk = fixed_mask[n];
    double fi[6], ri[6], zi[6], kx[6];
    ld6(f, n, fi);
    if (warm) ld6(Kx0, n, kx);
#pragma unroll
    for (int a = 0; a < 6; ++a) {
      if ((mk >> a) & 1) fi[a] = 0.0;
      ri[a] = warm ? fi[a] - kx[a] : fi[a];
    }
    st6(fbc, n, fi);
    if (!warm) {
      const double zero[6] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
      st6(x, n, zero);
    }
    st6(r, n, ri);
    block_apply(binv, n_nodes, n, ri, zi);
    st6(z, n, zi);
    st6(p, n, zi);
#pragma unroll
    for (int a = 0; a < 6; ++a) {
      v[0] += fi[a] * fi[a];
      v[1] += ri[a] * zi[a];
      v[2] += ri[a] * ri[a];
    }
  }
  if (grid_sum<3>(v, partial, &st->ticket[2], sm) && threadIdx.x == 0) {
    st->ff = v[0];
    st->rz = v[1];
    st->rr = v[2];
    st->iter = 0;
    st->status = SSO_OK;
    st->done = (v[2] <= st->tol2 * v[0] || v[0] == 0.0) ? 1 : 0;
    st->tol2 = st->tol2 * v[0];
    st->alpha = st->beta = 0.0;
    st->rr_ref = v[2];
  }
}

// x += alpha p, r -= alpha q, z = M^-1 r (stored); r^T z, r^T r -> beta, convergence (update epilogue)
__global__ void __launch_bounds__(256) cg_update_block_kernel(int n_nodes, const double* __restrict__ binv,
                                                              double* __restrict__ x, double* __restrict__ r,
                                                              const double* __restrict__ p,
                                                              const double* __restrict__ q, double* __restrict__ z,
                                                              double* __restrict__ partial, CgState* st,
                                                              BatchStrides bs) {
  __shared__ double sm[64];
  {
    const int bd = blockIdx.y;
    binv += (int64_t)bd * 21 * n_nodes;
    x += bd * bs.dof;
    r += bd * bs.dof;
    p += bd * bs.dof;
    q += bd * bs.dof;
    z += bd * bs.dof;
    partial += bd * bs.partial;
    st += bd;
  }
  if (st->done) return;
  const double alpha = st->alpha;
  double v[2] = {0.0, 0.0};
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t n = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; n < n_nodes; n += stride) {
    double xi[6], ri[6], pi[6], qi[6], zi[6];
    ld6(x, n, xi);
    ld6(r, n, ri);
    ld6(p, n, pi);
    ld6(q, n, qi);
#pragma unroll
    for (int a = 0; a < 6; ++a) {
      xi[a] += alpha * pi[a];
      ri[a] -= alpha * qi[a];
    }
    st6(x, n, xi);
    st6(r, n, ri);
    block_apply(binv, n_nodes, n, ri, zi);
    st6(z, n, zi);
#pragma unroll
    for (int a = 0; a < 6; ++a) {
      v[0] += ri[a] * zi[a];
      v[1] += ri[a] * ri[a];
    }
  }
  if (grid_sum<2>(v, partial, &st->ticket[1], sm) && threadIdx.x == 0) {
    const double rz_new = v[0];
    st->beta = rz_new / st->rz;
    st->rz_prev = st->rz;
    st->rz = rz_new;
    st->rr = v[1];
    st->iter += 1;
    lz_record(st, st->alpha, st->beta);
    if (v[1] <= st->tol2) {
      st->done = 1;
      st->status = SSO_OK;
    } else if (st->iter >= st->max_iter) {
      st->done = 1;
      st->status = SSO_E_NOT_CONVERGED;
    }
  }
}

// p = z + beta p
__global__ void __launch_bounds__(256) cg_pupdate_z_kernel(int ndof, const double* __restrict__ z,
                                                           double* __restrict__ p, const CgState* st,
                                                           BatchStrides bs) {
  {
    const int bd = blockIdx.y;
    z += bd * bs.dof;
    p += bd * bs.dof;
    st += bd;
  }
  if (st->done) return;
  const double beta = st->beta;
  const int64_t n2 = ndof / 2;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const double2* __restrict__ z2 = reinterpret_cast<const double2*>(z);
  double2* __restrict__ p2 = reinterpret_cast<double2*>(p);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n2; i += stride) {
    const double2 zi = z2[i];
    double2 pi = p2[i];
    pi.x = __fma_rn(beta, pi.x, zi.x);  // the rounding of the fused form
    pi.y = __fma_rn(beta, pi.y, zi.y);
    p2[i] = pi;
  }
}

// Fused form of cg_update_block + cg_pupdate_z (one part, B <= cg_fused_grid()):
// x += alpha p, r -= alpha q, z = M^-1 r with r^T z, r^T r over the grid, the grid
// barrier of cg_fused.cuh, then p_next = z + beta p into the other p buffer, z kept
// in registers for the first FB_ITEMS nodes of each thread (no z round trip).
constexpr int FB_ITEMS = 3;

__global__ void __launch_bounds__(256, 2) cg_update_block_fused_kernel(
    int n_nodes, const double* __restrict__ binv, double* __restrict__ x, double* __restrict__ r,
    const double* __restrict__ p, const double* __restrict__ q, double* __restrict__ pn,
    double* __restrict__ partial, CgState* st, BatchStrides bs) {
  __shared__ double sm[64];
  {
    const int bd = blockIdx.y;
    binv += (int64_t)bd * 21 * n_nodes;
    x += bd * bs.dof;
    r += bd * bs.dof;
    p += bd * bs.dof;
    q += bd * bs.dof;
    pn += bd * bs.dof;
    partial += bd * bs.partial;
    st += bd;
  }
  if (st->done) return;
  const double rz_old = st->rz;  // before CTA 0 rewrites it
  const long long iter_old = st->iter;
  double alpha, pqv;
  if (!cg_fused_alpha(partial + PQ_OFF, st, sm, rz_old, alpha, pqv)) return;
  double v[2] = {0.0, 0.0};
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t n0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  double zk[FB_ITEMS][6], pk[FB_ITEMS][6];
  auto step = [&](int64_t n, double (&zi)[6], double (&pi)[6]) {
    double xi[6], ri[6], qi[6];
    ld6(x, n, xi);
    ld6(r, n, ri);
    ld6(p, n, pi);
    ld6(q, n, qi);
#pragma unroll
    for (int a = 0; a < 6; ++a) {
      xi[a] += alpha * pi[a];
      ri[a] -= alpha * qi[a];
    }
    st6(x, n, xi);
    st6(r, n, ri);
    block_apply(binv, n_nodes, n, ri, zi);
#pragma unroll
    for (int a = 0; a < 6; ++a) {
      v[0] += ri[a] * zi[a];
      v[1] += ri[a] * ri[a];
    }
  };
#pragma unroll
  for (int k = 0; k < FB_ITEMS; ++k)
    if (n0 + k * stride < n_nodes) step(n0 + k * stride, zk[k], pk[k]);
  for (int64_t n = n0 + FB_ITEMS * stride; n < n_nodes; n += stride) {
    double zi[6], pi[6];
    step(n, zi, pi);
  }
  if (!cg_fused_allreduce(v, partial, &st->arrive, sm)) {
    if (threadIdx.x == 0) {
      st->status = SSO_E_CUDA;
      st->done = 1;
    }
    return;
  }
  double beta;
  if (!cg_fused_step(v, st, rz_old, iter_old, alpha, pqv, beta)) return;
#pragma unroll
  for (int k = 0; k < FB_ITEMS; ++k) {
    const int64_t n = n0 + k * stride;
    if (n < n_nodes) {
      double o[6];
#pragma unroll
      for (int a = 0; a < 6; ++a) o[a] = __fma_rn(beta, pk[k][a], zk[k][a]);
      st6(pn, n, o);
    }
  }
  for (int64_t n = n0 + FB_ITEMS * stride; n < n_nodes; n += stride) {
    double ri[6], pi[6], zi[6], o[6];
    ld6(r, n, ri);
    ld6(p, n, pi);
    block_apply(binv, n_nodes, n, ri, zi);
#pragma unroll
    for (int a = 0; a < 6; ++a) o[a] = __fma_rn(beta, pi[a], zi[a]);
    st6(pn, n, o);
  }
}

// p_out = z + beta p_in after a residual replacement of the fused form (z from
// cg_replace_block_kernel)
__global__ void __launch_bounds__(256) cg_pfix_z_kernel(int ndof, const double* __restrict__ z,
                                                        const double* __restrict__ pin,
                                                        double* __restrict__ pout, const CgState* st,
                                                        BatchStrides bs) {
  {
    const int bd = blockIdx.y;
    z += bd * bs.dof;
    pin += bd * bs.dof;
    pout += bd * bs.dof;
    st += bd;
  }
  if (st->done || !st->pfix) return;
  const double beta = st->beta;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < ndof; i += stride)
    pout[i] = __fma_rn(beta, pin[i], z[i]);
}

// Residual replacement (designs selected by cg_check): r = f_bc - K x, z = M^-1 r (replace epilogue)
__global__ void __launch_bounds__(256) cg_replace_block_kernel(int n_nodes, const double* __restrict__ fbc,
                                                               const double* __restrict__ Kx,
                                                               const double* __restrict__ binv,
                                                               double* __restrict__ r, double* __restrict__ z,
                                                               double* __restrict__ partial, CgState* st, int mode,
                                                               BatchStrides bs) {
  __shared__ double sm[64];
  {
    const int bd = blockIdx.y;
    fbc += bd * bs.dof;
    Kx += bd * bs.dof;
    binv += (int64_t)bd * 21 * n_nodes;
    r += bd * bs.dof;
    z += bd * bs.dof;
    partial += bd * bs.partial;
    st += bd;
  }
  if (!st->act) return;
  double v[2] = {0.0, 0.0};
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t n = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; n < n_nodes; n += stride) {
    double fi[6], ki[6], ri[6], zi[6];
    ld6(fbc, n, fi);
    ld6(Kx, n, ki);
#pragma unroll
    for (int a = 0; a < 6; ++a) ri[a] = fi[a] - ki[a];
    st6(r, n, ri);
    block_apply(binv, n_nodes, n, ri, zi);
    st6(z, n, zi);
#pragma unroll
    for (int a = 0; a < 6; ++a) {
      v[0] += ri[a] * zi[a];
      v[1] += ri[a] * ri[a];
    }
  }
  if (grid_sum<2>(v, partial, &st->ticket[1], sm) && threadIdx.x == 0) {
    st->rz = v[0];
    st->rr = v[1];
    st->rr_ref = v[1];
    st->beta = (mode == REPL_FINAL || st->act == 2) ? 0.0 : v[0] / st->rz_prev;
    st->act = 0;
    st->pfix = 1;
  }
}

int node_grid(int64_t n, int B) {
  const int64_t need = (n + 255) / 256;
  return (int)std::max<int64_t>(1, std::min<int64_t>(need, (int64_t)cg_grid() / B));
}

}  // namespace

void launch_block_inverse(cudaStream_t s, int n_nodes, const int64_t* node_ptr, const int32_t* node_col,
                          const double* vals, int layout, double* binv, DevFlags* flags, const BatchStrides& bs) {
  if (n_nodes <= 0) return;
  block_inverse_kernel<<<dim3((n_nodes + 127) / 128, bs.B), 128, 0, s>>>(n_nodes, node_ptr, node_col, vals, layout,
                                                                         binv, flags, bs);
  SSO_POST_LAUNCH("block_inverse_kernel");
}

void launch_cg_init_block(cudaStream_t s, int n_nodes, const double* f, const uint8_t* fixed_mask,
                          const double* binv, double* fbc, double* x, double* r, double* p, double* z,
                          double* partial, CgState* st, int warm, const double* Kx0, const BatchStrides& bs) {
  cg_init_block_kernel<<<dim3(node_grid(n_nodes, bs.B), bs.B), 256, 0, s>>>(n_nodes, f, fixed_mask, binv, fbc, x,
                                                                             r, p, z, partial, st, warm, Kx0, bs);
  SSO_POST_LAUNCH("cg_init_block_kernel");
}

void launch_cg_update_block(cudaStream_t s, int n_nodes, const double* binv, double* x, double* r,
                            const double* p, const double* q, double* z, double* partial, CgState* st,
                            const BatchStrides& bs) {
  cg_update_block_kernel<<<dim3(node_grid(n_nodes, bs.B), bs.B), 256, 0, s>>>(n_nodes, binv, x, r, p, q, z,
                                                                               partial, st, bs);
  SSO_POST_LAUNCH("cg_update_block_kernel");
}

void launch_cg_pupdate_z(cudaStream_t s, int ndof, const double* z, double* p, CgState* st,
                         const BatchStrides& bs) {
  const int64_t need = ((int64_t)ndof / 2 + 255) / 256;
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(need, (int64_t)cg_grid() / bs.B));
  cg_pupdate_z_kernel<<<dim3(grid, bs.B), 256, 0, s>>>(ndof, z, p, st, bs);
  SSO_POST_LAUNCH("cg_pupdate_z_kernel");
}

int cg_block_fused_grid() {
  static int g = -1;
  if (g < 0) {
    int occ = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, cg_update_block_fused_kernel, 256, 0) != cudaSuccess)
      occ = 0;
    g = std::min(occ, 2) * (cg_grid() / 4);
  }
  return g;
}

void launch_cg_update_block_fused(cudaStream_t s, int n_nodes, const double* binv, double* x, double* r,
                                  const double* p, const double* q, double* pn, double* partial, CgState* st,
                                  const BatchStrides& bs) {
  const int64_t need = ((int64_t)n_nodes + 255) / 256;
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(need, cg_block_fused_grid() / bs.B));
  const cudaError_t e = launch_cooperative(cg_update_block_fused_kernel, dim3(grid, bs.B), dim3(256), s, n_nodes,
                                           binv, x, r, p, q, pn, partial, st, bs);
  SSO_POST_LAUNCH_RC("cg_update_block_fused_kernel", e);
}

void launch_cg_pfix_z(cudaStream_t s, int ndof, const double* z, const double* pin, double* pout,
                      const CgState* st, const BatchStrides& bs) {
  const int grid = node_grid(ndof / 6, bs.B);
  cg_pfix_z_kernel<<<dim3(grid, bs.B), 256, 0, s>>>(ndof, z, pin, pout, st, bs);
  SSO_POST_LAUNCH("cg_pfix_z_kernel");
}

void launch_cg_replace_block(cudaStream_t s, int n_nodes, const double* fbc, const double* Kx, const double* binv,
                             double* r, double* z, double* partial, CgState* st, int mode, const BatchStrides& bs) {
  cg_replace_block_kernel<<<dim3(node_grid(n_nodes, bs.B), bs.B), 256, 0, s>>>(n_nodes, fbc, Kx, binv, r, z,
                                                                                partial, st, mode, bs);
  SSO_POST_LAUNCH("cg_replace_block_kernel");
}

}  // namespace sso
