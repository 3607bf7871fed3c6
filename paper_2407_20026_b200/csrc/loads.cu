// Design-dependent area loads (Eq. 6 with
// df/dp != 0; reading c17).  Every quad carries a load per unit area (q_e + w_e t_e)
// in the direction d, lumped equally to its 4 nodes with
//     A_e = 1/2 |(X3 - X1) x (X4 - X2)|,   f_n[0:3] += d (q_e + w_e t_e) A_e / 4.
// The gradient term v^T df/dp (v = 2 s u for the compliance, lambda for a general
// objective) is added into the element-node slots of the gradient pass before the
// node reduction, so it inherits the pass's fixed summation order.
#include "sso_internal.h"

namespace sso {

namespace {

__device__ __forceinline__ void quad_diagonals(const double* __restrict__ gx, const double* __restrict__ gy,
                                               const double* __restrict__ gz, const int32_t* nd, double d1[3],
                                               double d2[3]) {
  d1[0] = gx[nd[2]] - gx[nd[0]];
  d1[1] = gy[nd[2]] - gy[nd[0]];
  d1[2] = gz[nd[2]] - gz[nd[0]];
  d2[0] = gx[nd[3]] - gx[nd[1]];
  d2[1] = gy[nd[3]] - gy[nd[1]];
  d2[2] = gz[nd[3]] - gz[nd[1]];
}

// a[q] = (q_e + w_e t_e) A_e / 4 (per node of the quad, before the direction)
__global__ void __launch_bounds__(256) area_load_elem_kernel(
    int n_quads, const double* __restrict__ gx, const double* __restrict__ gy, const double* __restrict__ gz,
    const int32_t* __restrict__ conn, const double* __restrict__ gt, const double* __restrict__ lq,
    const double* __restrict__ lw, double* __restrict__ a, BatchStrides bs) {
  const int bd = blockIdx.y;
  gx += bd * bs.node;
  gy += bd * bs.node;
  gz += bd * bs.node;
  gt += bd * bs.quad;
  a += bd * bs.quad;
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < n_quads;
       q += (int64_t)gridDim.x * blockDim.x) {
    int32_t nd[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) nd[k] = __ldg(conn + 4 * q + k);
    double d1[3], d2[3];
    quad_diagonals(gx, gy, gz, nd, d1, d2);
    const double c0 = d1[1] * d2[2] - d1[2] * d2[1];
    const double c1 = d1[2] * d2[0] - d1[0] * d2[2];
    const double c2 = d1[0] * d2[1] - d1[1] * d2[0];
    const double area = 0.5 * sqrt(c0 * c0 + c1 * c1 + c2 * c2);
    a[q] = (lq[q] + lw[q] * gt[q]) * area / 4.0;
  }
}

// f_n[0:3] += d * sum over the node's incident quads (ascending element order) of a[q]
__global__ void __launch_bounds__(256) area_load_node_kernel(
    int n_nodes, int n_beams, const int64_t* __restrict__ inc_ptr, const int32_t* __restrict__ inc_slot,
    const double* __restrict__ a, double d0, double d1, double d2, double* __restrict__ f, BatchStrides bs) {
  const int bd = blockIdx.y;
  a += bd * bs.quad;
  f += bd * bs.dof;
  for (int64_t n = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; n < n_nodes;
       n += (int64_t)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int64_t k = inc_ptr[n]; k < inc_ptr[n + 1]; ++k) {
      const int64_t sl = inc_slot[k] - 2 * (int64_t)n_beams;
      if (sl >= 0) s += a[sl >> 2];
    }
    f[6 * n + 0] += d0 * s;
    f[6 * n + 1] += d1 * s;
    f[6 * n + 2] += d2 * s;
  }
}

// slot[quad q, node k] += coef (d . sum_k v_k) (q_e + w_e t_e)/4 dA_e/dX_k;  dt[q] += coef (d . sum v) w_e A_e/4
__global__ void __launch_bounds__(256) area_load_grad_kernel(
    int n_beams, int n_quads, const double* __restrict__ gx, const double* __restrict__ gy,
    const double* __restrict__ gz, const int32_t* __restrict__ conn, const double* __restrict__ gt,
    const double* __restrict__ lq, const double* __restrict__ lw, double dir0, double dir1, double dir2,
    const double* __restrict__ v, double coef, double* __restrict__ slot_partial, double* __restrict__ dt,
    BatchStrides bs) {
  const int bd = blockIdx.y;
  gx += bd * bs.node;
  gy += bd * bs.node;
  gz += bd * bs.node;
  gt += bd * bs.quad;
  v += bd * bs.dof;
  slot_partial += bd * bs.slot;
  dt += bd * bs.quad;
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < n_quads;
       q += (int64_t)gridDim.x * blockDim.x) {
    int32_t nd[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) nd[k] = __ldg(conn + 4 * q + k);
    double U = 0.0;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const double* vk = v + 6 * (int64_t)nd[k];
      U += dir0 * vk[0] + dir1 * vk[1] + dir2 * vk[2];
    }
    const double g = coef * U;
    double d1[3], d2[3];
    quad_diagonals(gx, gy, gz, nd, d1, d2);
    double c[3] = {d1[1] * d2[2] - d1[2] * d2[1], d1[2] * d2[0] - d1[0] * d2[2], d1[0] * d2[1] - d1[1] * d2[0]};
    const double cn = sqrt(c[0] * c[0] + c[1] * c[1] + c[2] * c[2]);
    const double area = 0.5 * cn;
    dt[q] += g * lw[q] * area / 4.0;
    if (cn > 0.0) {
      const double ic = 1.0 / cn;
      c[0] *= ic, c[1] *= ic, c[2] *= ic;
      // dA/dd1 = 1/2 d2 x c_hat, dA/dd2 = 1/2 c_hat x d1
      const double a1[3] = {0.5 * (d2[1] * c[2] - d2[2] * c[1]), 0.5 * (d2[2] * c[0] - d2[0] * c[2]),
                            0.5 * (d2[0] * c[1] - d2[1] * c[0])};
      const double a2[3] = {0.5 * (c[1] * d1[2] - c[2] * d1[1]), 0.5 * (c[2] * d1[0] - c[0] * d1[2]),
                            0.5 * (c[0] * d1[1] - c[1] * d1[0])};
      const double ga = g * (lq[q] + lw[q] * gt[q]) / 4.0;
      double* sp = slot_partial + (2 * (int64_t)n_beams + 4 * q) * 3;
#pragma unroll
      for (int x = 0; x < 3; ++x) {
        sp[0 * 3 + x] -= ga * a1[x];
        sp[2 * 3 + x] += ga * a1[x];
        sp[1 * 3 + x] -= ga * a2[x];
        sp[3 * 3 + x] += ga * a2[x];
      }
    }
  }
}

int grid_for(int64_t n) { return (int)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 148 * 16)); }

}  // namespace

void launch_area_load(cudaStream_t s, int n_own, int n_beams, int n_quads, const double* x, const double* y,
                      const double* z, const int32_t* conn, const double* t, const double* lq, const double* lw,
                      const double dir[3], const int64_t* inc_ptr, const int32_t* inc_slot, double* a, double* f,
                      const BatchStrides& bs) {
  if (n_quads > 0) {
    area_load_elem_kernel<<<dim3(grid_for(n_quads), bs.B), 256, 0, s>>>(n_quads, x, y, z, conn, t, lq, lw, a, bs);
    SSO_POST_LAUNCH("area_load_elem_kernel");
  }
  if (n_own > 0) {
    area_load_node_kernel<<<dim3(grid_for(n_own), bs.B), 256, 0, s>>>(n_own, n_beams, inc_ptr, inc_slot, a, dir[0],
                                                                      dir[1], dir[2], f, bs);
    SSO_POST_LAUNCH("area_load_node_kernel");
  }
}

void launch_area_load_grad(cudaStream_t s, int n_beams, int n_quads, const double* x, const double* y,
                           const double* z, const int32_t* conn, const double* t, const double* lq,
                           const double* lw, const double dir[3], const double* v, double coef,
                           double* slot_partial, double* dt, const BatchStrides& bs) {
  if (n_quads <= 0) return;
  area_load_grad_kernel<<<dim3(grid_for(n_quads), bs.B), 256, 0, s>>>(
      n_beams, n_quads, x, y, z, conn, t, lq, lw, dir[0], dir[1], dir[2], v, coef, slot_partial, dt, bs);
  SSO_POST_LAUNCH("area_load_grad_kernel");
}

}  // namespace sso
