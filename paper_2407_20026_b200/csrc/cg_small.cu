// Cluster-resident point-Jacobi PCG for small models (sm_100a): a chunk of CG iterations of
// each design in ONE thread-block cluster.
//
// PAPER.md:71-74 (Eq. 1) solved by PCG in its single-reduction (Chronopoulos-Gear) form, the
// form the partitioned handles use (cg_sr.cu, reading c21): with u = M^-1 r and w = K u,
//   gamma = r^T u, delta = u^T w, beta = gamma / gamma_old,
//   alpha = gamma / (delta - beta gamma / alpha_old)   (= gamma / p^T K p),
//   p = u + beta p, s = w + beta s (= K p), x += alpha p, r -= alpha s,
// the same alpha_k, beta_k as the classic recurrence in exact arithmetic (and the same Lanczos
// record), with ONE reduction per iteration.  For the latency configurations (C1: 150 DOF, C2:
// 2 646 DOF) the two-kernel iteration costs ~10 us, almost all of it launch and drain latency
// of kernels with < 1 us of work.  Here one cluster of up to 16 CTAs owns a design for the
// whole chunk:
//   * CTA c of the cluster owns nodes [c npt, (c + 1) npt); thread rows keep x, r, dinv, p, s
//     and u of their DOFs in registers across iterations;
//   * the 54 values of each row (storage-3 own run and pulled blocks) and the addresses of its
//     neighbours' u rows are staged in shared memory once per chunk; u lives in the owners'
//     shared memory: w = K u of a row reads its neighbours' u through distributed shared memory
//     (DSMEM, ~215 cycles) -- no global memory access inside the iteration;
//   * two cluster barriers per iteration: the CTAs' partials (u^T w, r^T u, r^T r), pushed into
//     every CTA's table by remote stores and summed in rank order (identical alpha, beta and
//     convergence decision in every CTA -- a divergence would desynchronise the barriers;
//     cluster rank 0 records the state), then the publication of u.
// Designs of a batch are independent clusters (grid = B clusters): no grid-wide co-residency.
// Models up to CL_MAX_CS x CL_MAX_NPT = 1 152 nodes whose nodes all fit the pull descriptor.
// Between chunks x, r, p and s (in the fused path's second p buffer) persist in global memory;
// a fresh solve or a replaced residual (cg_replace sets pfix) restarts the recurrence (beta = 0).
#include <cooperative_groups.h>

#include "sso_internal.h"

namespace cg = cooperative_groups;

namespace sso {

namespace {

constexpr int CL_THREADS = 256;
constexpr int CL_RMAX = 2;          // rows per thread: 6 npt <= CL_THREADS CL_RMAX
constexpr int CL_MAX_NPT = 72;        // 6 npt <= CL_THREADS CL_RMAX rows; staged smem <= 227 KB
constexpr int CL_MAX_CS = 16;       // non-portable cluster size
constexpr int CL_DESC = 16;         // int32 per node descriptor (pcg.cu PULL_DESC)
constexpr int CL_VALS = 54;         // the row's values of its <= 9 blocks (6 each)
static_assert(CL_RMAX * CL_THREADS >= 6 * CL_MAX_NPT, "rows per CTA");

// cluster barrier; a single-CTA "cluster" (small models) needs only the CTA barrier
__device__ __forceinline__ void csync(const cg::cluster_group& cl, int CS) {
  if (CS == 1)
    __syncthreads();
  else
    cl.sync();
}

__device__ __forceinline__ void cl_block_sum3(double& v0, double& v1, double& v2, double* sm) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    v0 += __shfl_xor_sync(0xffffffffu, v0, o);
    v1 += __shfl_xor_sync(0xffffffffu, v1, o);
    v2 += __shfl_xor_sync(0xffffffffu, v2, o);
  }
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (lane == 0) {
    sm[3 * w] = v0;
    sm[3 * w + 1] = v1;
    sm[3 * w + 2] = v2;
  }
  __syncthreads();
  double t0 = 0.0, t1 = 0.0, t2 = 0.0;
  for (int i = 0; i < (int)(blockDim.x >> 5); ++i) {  // every thread, the same order
    t0 += sm[3 * i];
    t1 += sm[3 * i + 1];
    t2 += sm[3 * i + 2];
  }
  __syncthreads();
  v0 = t0;
  v1 = t1;
  v2 = t2;
}

// Staged operands of row rho (node n, row a) of this CTA: the 54 values of its <= 9 blocks
// (own upper blocks K_nm row a, then pulled blocks K_mn column a: the order of the pull
// kernel's general path) at kv[j 6 + c][rho] (zeros for unused blocks), and the
// shared::cluster address of each block's p_m row at km[j][rho].  Read once per chunk from the
// storage-3 records.
__device__ __forceinline__ void cl_stage(const cg::cluster_group& cl, int rho, int rows, int n, int a, int npt,
                                         int self, double* u_s, const int32_t* __restrict__ pdesc,
                                         const double* __restrict__ vals, double* kv, const double2** km) {
  const int32_t* Di = pdesc + CL_DESC * (int64_t)n;
  const int b0 = __ldg(Di), fl = __ldg(Di + 1);
  const int udeg = fl & 255, ldeg = (fl >> 8) & 255;  // fits (checked on the host)
#pragma unroll
  for (int j = 0; j < 9; ++j) {
    int m = -1, rec = b0;
    if (j < udeg) {
      m = __ldg(Di + 2 + j);
      rec = b0 + j;
    } else if (j < udeg + ldeg) {
      m = __ldg(Di + 2 + udeg + 2 * (j - udeg));
      rec = __ldg(Di + 3 + udeg + 2 * (j - udeg));
    }
    {  // p_m in its owner CTA's shared memory (this CTA's first row if unused)
      const int o = m < 0 ? self : m / npt;
      km[j * rows + rho] =
          reinterpret_cast<const double2*>(cl.map_shared_rank(u_s, o) + 6 * (m < 0 ? 0 : m - o * npt));
    }
    const double* bk = vals + PULL_BLOCK * (int64_t)rec;
#pragma unroll
    for (int c = 0; c < 6; ++c)
      kv[(6 * j + c) * rows + rho] = m < 0 ? 0.0 : __ldg(bk + (j < udeg ? rec_off(a, c) : rec_off(c, a)));
  }
}

// q of row rho from the staged operands; p_m from the owner CTA's shared memory (DSMEM)
__device__ __forceinline__ double cl_row(int rho, int rows, const double* kv, const double2* const* km) {
  double2 xv[9][3];
#pragma unroll
  for (int j = 0; j < 9; ++j) {
    const double2* xm = km[j * rows + rho];  // (the cluster barriers order these reads)
#pragma unroll
    for (int h = 0; h < 3; ++h) xv[j][h] = xm[h];
  }
  double y = 0.0;
#pragma unroll
  for (int j = 0; j < 9; ++j) {
    const double* kj = kv + 6 * j * rows + rho;
    double t = 0.0;
    t = fma(kj[0], xv[j][0].x, t);
    t = fma(kj[rows], xv[j][0].y, t);
    t = fma(kj[2 * rows], xv[j][1].x, t);
    t = fma(kj[3 * rows], xv[j][1].y, t);
    t = fma(kj[4 * rows], xv[j][2].x, t);
    t = fma(kj[5 * rows], xv[j][2].y, t);
    y += t;
  }
  return y;
}

__global__ void __launch_bounds__(CL_THREADS) cg_cluster_kernel(
    int n_nodes, int npt, int iters, const int32_t* __restrict__ pdesc, const double* __restrict__ vals,
    const double* __restrict__ dinv, double* __restrict__ x, double* __restrict__ r, double* __restrict__ p,
    double* __restrict__ s_vec, CgState* st, BatchStrides bs) {
  extern __shared__ __align__(16) double dsm[];
  __shared__ double sm[64];
  cg::cluster_group cl = cg::this_cluster();
  const int cr = (int)cl.block_rank(), CS = (int)cl.num_blocks();
  {  // design of a batch: one cluster per design
    const int bd = blockIdx.x / CS;
    vals += bd * bs.nnz;
    dinv += bd * bs.dof;
    x += bd * bs.dof;
    r += bd * bs.dof;
    p += bd * bs.dof;
    s_vec += bd * bs.dof;
    st += bd;
  }
  if (st->done) return;  // the same for every CTA of the cluster
  const int rows = 6 * npt;              // row capacity of a CTA
  double* u_s = dsm;                     // this CTA's u = M^-1 r rows [rows] (read by the cluster)
  // [c][0..2] u^T K u, r^T u, r^T r partials of cluster CTA c: every CTA pushes its partials
  // into every CTA's table (remote stores, no load latency), then sums its own table
  double* red = dsm + rows;
  double* kv = red + 4 * CL_MAX_CS;      // [54][rows] staged values
  const double2** km = reinterpret_cast<const double2**>(kv + CL_VALS * rows);  // [9][rows] p_m rows
  const bool writer = cr == 0 && threadIdx.x == 0;
  const int node0 = cr * npt;
  const int nrows = 6 * max(0, min(npt, n_nodes - node0));
  const int64_t g0 = 6 * (int64_t)node0;
  double xt[CL_RMAX], rt[CL_RMAX], dt[CL_RMAX], pt[CL_RMAX], sv[CL_RMAX], ut[CL_RMAX];
  // a fresh solve or a replaced residual (cg_replace set pfix) restarts the recurrence: beta = 0
  bool restart = st->iter == 0 || st->pfix;
#pragma unroll
  for (int k = 0; k < CL_RMAX; ++k) {
    const int rho = threadIdx.x + k * CL_THREADS;
    xt[k] = rt[k] = dt[k] = pt[k] = sv[k] = ut[k] = 0.0;
    if (rho < nrows) {
      xt[k] = x[g0 + rho];
      rt[k] = r[g0 + rho];
      dt[k] = dinv[g0 + rho];
      pt[k] = p[g0 + rho];
      sv[k] = s_vec[g0 + rho];
      ut[k] = __dmul_rn(dt[k], rt[k]);  // u = M^-1 r (the rounding of z in the fused path)
      u_s[rho] = ut[k];
      cl_stage(cl, rho, rows, node0 + rho / 6, rho % 6, npt, cr, u_s, pdesc, vals, kv, km);
    }
  }
  double gam_old = st->rz, alpha_old = st->alpha;
  long long iter = st->iter;
  const double tol2 = st->tol2;
  const long long max_iter = st->max_iter;
  // the Lanczos record (lz_record) with its bookkeeping in registers: no global read on the
  // writer's path inside the iteration
  double* const lz = st->lz;
  // a replaced residual restarts this recurrence (beta = 0) even where the classic path would
  // continue: a restarted CG is a new Lanczos sequence, so the record stops (as cg_check does
  // for its own restarts)
  const bool lz_cut = st->pfix && st->iter > 0;
  if (lz_cut && writer) st->lz_frozen = 1;
  const bool lz_on = lz && !st->lz_frozen && !lz_cut;
  const int lz_cap = st->lz_cap;
  int lz_n = st->lz_n;
  csync(cl, CS);
  for (int it = 0; it < iters; ++it) {
    // w = K u (rows), u^T w, r^T u, r^T r
    double wt[CL_RMAX];
    double a0 = 0.0, a1 = 0.0, a2 = 0.0;
#pragma unroll
    for (int k = 0; k < CL_RMAX; ++k) {
      const int rho = threadIdx.x + k * CL_THREADS;
      wt[k] = 0.0;
      if (rho < nrows) {
        wt[k] = cl_row(rho, rows, kv, km);
        a0 += ut[k] * wt[k];
        a1 += rt[k] * ut[k];
        a2 += rt[k] * rt[k];
      }
    }
    cl_block_sum3(a0, a1, a2, sm);
    if (threadIdx.x < CS) {
      double* t = cl.map_shared_rank(red, (int)threadIdx.x) + 4 * cr;
      t[0] = a0;
      t[1] = a1;
      t[2] = a2;
    }
    csync(cl, CS);  // partials in every table
    double delta = 0.0, gam = 0.0, rr = 0.0;
    for (int c = 0; c < CS; ++c) {  // rank order: the same totals in every CTA
      delta += red[4 * c];
      gam += red[4 * c + 1];
      rr += red[4 * c + 2];
    }
    // Lanczos record (lz_record) in the classic convention: (alpha_k, beta_k) with beta_k =
    // gamma_{k+1} / gamma_k, i.e. the previous iteration's alpha with this iteration's beta
    // (as cg_sr.cu); the last alpha of a run gets beta 0 (never formed)
    auto record = [&](double a, double b) {
      if (lz_on && lz_n < lz_cap) {
        lz[2 * lz_n] = a;
        lz[2 * lz_n + 1] = b;
        st->lz_n = ++lz_n;
      }
    };
    if (rr <= tol2) {  // r (the result of the last update) has converged
      if (writer) {
        if (!restart) record(alpha_old, 0.0);
        st->rr = rr;
        st->done = 1;
        st->status = SSO_OK;
      }
      break;
    }
    const double beta = restart ? 0.0 : gam / gam_old;
    const double pq = restart ? delta : delta - beta * gam / alpha_old;  // p^T K p of the new p
    if (!(pq > 0.0)) {
      if (writer) {
        if (!restart) record(alpha_old, 0.0);
        st->pq = pq;
        st->status = SSO_E_NOT_SPD;
        st->done = 1;
      }
      break;
    }
    const double alpha = gam / pq;
    const bool maxed = iter + 1 >= max_iter;
    if (writer) {
      if (!restart) record(alpha_old, beta);
      st->alpha = alpha;
      st->pq = pq;
      st->beta = beta;
      st->rz_prev = gam_old;
      st->rz = gam;
      st->rr = rr;
      st->iter = iter + 1;
      st->pfix = 0;
      if (maxed) {
        record(alpha, 0.0);
        st->done = 1;
        st->status = SSO_E_NOT_CONVERGED;
      }
    }
    // p = u + beta p, s = w + beta s (= K p), x += alpha p, r -= alpha s, u = M^-1 r
#pragma unroll
    for (int k = 0; k < CL_RMAX; ++k) {
      const int rho = threadIdx.x + k * CL_THREADS;
      if (rho < nrows) {
        pt[k] = __fma_rn(beta, pt[k], ut[k]);
        sv[k] = __fma_rn(beta, sv[k], wt[k]);
        xt[k] += alpha * pt[k];
        rt[k] -= alpha * sv[k];
        ut[k] = __dmul_rn(dt[k], rt[k]);
        u_s[rho] = ut[k];
      }
    }
    gam_old = gam;
    alpha_old = alpha;
    restart = false;
    ++iter;
    if (maxed) break;
    csync(cl, CS);  // u published; the partial tables free for the next iteration
  }
#pragma unroll
  for (int k = 0; k < CL_RMAX; ++k) {
    const int rho = threadIdx.x + k * CL_THREADS;
    if (rho < nrows) {
      x[g0 + rho] = xt[k];
      r[g0 + rho] = rt[k];
      p[g0 + rho] = pt[k];
      s_vec[g0 + rho] = sv[k];
    }
  }
  csync(cl, CS);  // no CTA leaves while a peer may still read its shared memory
}

int cl_npt(int n_nodes) {  // nodes per CTA: one CTA when the model fits it, else >= 16 per CTA
  if (n_nodes <= CL_MAX_NPT) return n_nodes;
  return std::max(16, (n_nodes + CL_MAX_CS - 1) / CL_MAX_CS);
}

size_t cl_smem(int npt) {
  return (size_t)6 * npt * (sizeof(double) * (1 + CL_VALS) + sizeof(void*) * 9) + sizeof(double) * 4 * CL_MAX_CS;
}

}  // namespace

static void cl_attributes() {
  static uint64_t attr_mask = 0;
  if (first_on_device(attr_mask)) {
    cudaFuncSetAttribute(cg_cluster_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaFuncSetAttribute(cg_cluster_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)cl_smem(CL_MAX_NPT));
  }
}

bool cg_small_fits(int n_nodes) {
  if (n_nodes <= 0 || cl_npt(n_nodes) > CL_MAX_NPT) return false;
  // the device must be able to place the cluster (its CTAs on SMs of one GPC)
  cl_attributes();
  const int npt = cl_npt(n_nodes), cs = (n_nodes + npt - 1) / npt;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(cs);
  cfg.blockDim = dim3(CL_THREADS);
  cfg.dynamicSmemBytes = cl_smem(npt);
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = cs;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  int nclusters = 0;
  if (cudaOccupancyMaxActiveClusters(&nclusters, cg_cluster_kernel, &cfg) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return nclusters >= 1;
}

void launch_cg_small(cudaStream_t s, int n_nodes, int iters, const int32_t* pdesc, const double* vals,
                     const double* dinv, double* x, double* r, double* p, double* s_vec, CgState* st,
                     const BatchStrides& bs) {
  const int npt = cl_npt(n_nodes);
  const int cs = (n_nodes + npt - 1) / npt;
  const size_t smem = cl_smem(npt);
  cl_attributes();
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(cs * bs.B);
  cfg.blockDim = dim3(CL_THREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = cs;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  const cudaError_t e = cudaLaunchKernelEx(&cfg, cg_cluster_kernel, n_nodes, npt, iters, pdesc, vals, dinv, x, r,
                                           p, s_vec, st, bs);
  SSO_POST_LAUNCH_RC("cg_cluster_kernel", e);
}

}  // namespace sso
