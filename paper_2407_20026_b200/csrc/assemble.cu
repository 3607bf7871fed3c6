// A2 — atomic-free segmented-sum assembly + supports + Jacobi diagonal (sm_100a).
//
// the global K is the sum of all element matrices scattered to
// their global positions (JAX-SSO: vmap + BCOO with summed duplicates).  Here
// the sum is a GATHER: each node owns a contiguous run of 36 deg(n) CSR values
// (its six scalar rows), and every value is the sum of the staged element
// blocks listed for its node-block, in ascending element order (reading c8).
// No atomics -> bit-reproducible.  Supports (Eq. 2-3 with b = 0,
// reading c1) by symmetric elimination: a value whose row or column DOF is
// fixed is zeroed unless it is a diagonal entry (kept; 1.0 if it is 0).  The
// Jacobi inverse diagonal dinv = 1 / K_bc[d][d] is produced in the same pass;
// a free DOF with a non-positive diagonal is flagged SINGULAR.
//
// Mapping: one warp per node, lanes striding over the node's 36 deg values;
// the stores are fully coalesced; the staged reads are 6-double runs.
#include <climits>

#include "sso_internal.h"

namespace sso {

namespace {

__global__ void __launch_bounds__(256) assemble_kernel(
    int n_nodes, const int64_t* __restrict__ node_ptr, const int32_t* __restrict__ node_col,
    const int64_t* __restrict__ contrib_ptr, const int32_t* __restrict__ contrib,
    const double* __restrict__ stage, const uint8_t* __restrict__ fixed_mask,
    double* __restrict__ vals, double* __restrict__ dinv, DevFlags* flags, BatchStrides bs, int cm) {
  {  // design of a batch (blockIdx.y)
    const int bd = blockIdx.y;
    stage += bd * bs.stage;
    vals += bd * bs.nnz;
    dinv += bd * bs.dof;
    flags += bd;
  }
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t n = warp; n < n_nodes; n += nwarps) {
    const int64_t b0 = node_ptr[n];
    const int deg = (int)(node_ptr[n + 1] - b0);
    const int rowlen = 6 * deg;
    const int total = 36 * deg;
    const uint8_t mrow = fixed_mask[n];
    // run layout: row-major (a, rem) runs, or (cm) one PULL_BLOCK record per block (rec_off)
    double* out = vals + (cm ? PULL_BLOCK : 36) * b0;
    for (int v = lane; v < total; v += 32) {
      const int a = cm ? v % 6 : v / rowlen;
      const int rem = cm ? v / 6 : v - a * rowlen;
      const int k = rem / 6;
      const int b = rem - 6 * k;
      const int dst = cm ? PULL_BLOCK * k + rec_off(a, b) : v;
      const int64_t blk = b0 + k;
      const int m = node_col[blk];
      double s = 0.0;
      const int64_t c1 = contrib_ptr[blk + 1];
      for (int64_t c = contrib_ptr[blk]; c < c1; ++c)
        s += stage[(int64_t)contrib[c] * 36 + 6 * a + b];
      const bool diag = (m == n) && (a == b);
      const bool rfix = (mrow >> a) & 1;
      const bool cfix = (fixed_mask[m] >> b) & 1;
      if (rfix || cfix) {
        if (diag) {
          if (s == 0.0) s = 1.0;
        } else {
          s = 0.0;
        }
      }
      out[dst] = s;
      if (diag) {
        if (!(s > 0.0)) atomicMin(&flags->singular_dof, (int)(6 * n + a));
        dinv[6 * n + a] = 1.0 / s;
      }
    }
  }
}

}  // namespace

void launch_assemble(cudaStream_t s, int n_nodes, const int64_t* node_ptr,
                     const int32_t* node_col, const int64_t* contrib_ptr,
                     const int32_t* contrib, const double* stage, const uint8_t* fixed_mask,
                     double* vals, double* dinv, DevFlags* flags, const BatchStrides& bs, int cm) {
  if (n_nodes <= 0) return;
  const int warps_per_cta = 8;
  int64_t need = ((int64_t)n_nodes + warps_per_cta - 1) / warps_per_cta;
  const dim3 grid((unsigned)std::max<int64_t>(1, std::min<int64_t>(need, (int64_t)cg_grid() * 4 / bs.B)), bs.B);
  assemble_kernel<<<grid, 32 * warps_per_cta, 0, s>>>(n_nodes, node_ptr, node_col, contrib_ptr,
                                                       contrib, stage, fixed_mask, vals, dinv,
                                                       flags, bs, cm);
  SSO_POST_LAUNCH("assemble_kernel");
}

}  // namespace sso
