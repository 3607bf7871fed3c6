// Hat filter of sensitivities:
//   out_i = sum_j w_ij in_j / sum_j w_ij,  w_ij = max(0, r - |X_i - X_j|)
// over node coordinates or element centroids (reading c16).  Matrix-free: the
// points are sorted into cubic cells of edge >= r (host), and one warp per output
// point walks the 27 neighbouring cells, lanes striding over the cell's points,
// with a fixed-order warp reduction (deterministic).
#include "sso_internal.h"

namespace sso {

namespace {

__device__ __forceinline__ double wsum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__global__ void __launch_bounds__(256) hat_filter_kernel(
    int n, int ncomp, const double* __restrict__ px, const double* __restrict__ py,
    const double* __restrict__ pz, const int32_t* __restrict__ cell_of, const int32_t* __restrict__ perm,
    const int64_t* __restrict__ cell_start, int gx, int gy, int gz, double radius,
    const double* __restrict__ in, double* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t i = warp; i < n; i += nw) {
    // px/py/pz are in sorted order; perm[k] = original index of sorted point k
    const int32_t si = cell_of[i];  // sorted position of point i
    const double xi = px[si], yi = py[si], zi = pz[si];
    const int32_t c = __ldg(cell_of + n + i);  // cell id of point i
    const int cx = c % gx, cy = (c / gx) % gy, cz = c / (gx * gy);
    double num0 = 0.0, num1 = 0.0, num2 = 0.0, den = 0.0;
    for (int dz = -1; dz <= 1; ++dz) {
      const int zz = cz + dz;
      if (zz < 0 || zz >= gz) continue;
      for (int dy = -1; dy <= 1; ++dy) {
        const int yy = cy + dy;
        if (yy < 0 || yy >= gy) continue;
        for (int dx = -1; dx <= 1; ++dx) {
          const int xx = cx + dx;
          if (xx < 0 || xx >= gx) continue;
          const int64_t cc = ((int64_t)zz * gy + yy) * gx + xx;
          for (int64_t k = cell_start[cc] + lane; k < cell_start[cc + 1]; k += 32) {
            const double ddx = px[k] - xi, ddy = py[k] - yi, ddz = pz[k] - zi;
            const double w = radius - sqrt(ddx * ddx + ddy * ddy + ddz * ddz);
            if (w > 0.0) {
              const int32_t j = perm[k];
              den += w;
              num0 += w * in[j];
              if (ncomp > 1) num1 += w * in[(int64_t)n + j];
              if (ncomp > 2) num2 += w * in[2 * (int64_t)n + j];
            }
          }
        }
      }
    }
    den = wsum(den);
    num0 = wsum(num0);
    if (ncomp > 1) num1 = wsum(num1);
    if (ncomp > 2) num2 = wsum(num2);
    if (lane == 0) {
      out[i] = num0 / den;
      if (ncomp > 1) out[(int64_t)n + i] = num1 / den;
      if (ncomp > 2) out[2 * (int64_t)n + i] = num2 / den;
    }
  }
}

}  // namespace

void launch_hat_filter(cudaStream_t s, int n, int ncomp, const double* px, const double* py,
                       const double* pz, const int32_t* cell_of, const int32_t* perm,
                       const int64_t* cell_start, int gx, int gy, int gz, double radius,
                       const double* in, double* out) {
  if (n <= 0) return;
  int64_t need = ((int64_t)n + 7) / 8;
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(need, (int64_t)cg_grid() * 2));
  hat_filter_kernel<<<grid, 256, 0, s>>>(n, ncomp, px, py, pz, cell_of, perm, cell_start, gx, gy, gz, radius,
                                         in, out);
  SSO_POST_LAUNCH("hat_filter_kernel");
}

}  // namespace sso
