// Small fp64 helpers shared by the element kernels (elements.cu, assemble_fused.cu).
#pragma once

namespace sso {
namespace shell {

__device__ __forceinline__ void cross3(const double* a, const double* b, double* c) {
  c[0] = a[1] * b[2] - a[2] * b[1];
  c[1] = a[2] * b[0] - a[0] * b[2];
  c[2] = a[0] * b[1] - a[1] * b[0];
}
__device__ __forceinline__ double dot3(const double* a, const double* b) {
  return a[0] * b[0] + a[1] * b[1] + a[2] * b[2];
}

// K_g = R6^T K' R6 where K' = W_i^T K W_j (local, in place) and R rows = (e1, e2, e3).
__device__ __forceinline__ void transform_block(double (&K)[6][6], const double (&R)[3][3],
                                                double hi, double hj) {
  // K W_j: col th_x += h_j col v ; col th_y -= h_j col u
#pragma unroll
  for (int a = 0; a < 6; ++a) {
    K[a][3] += hj * K[a][1];
    K[a][4] -= hj * K[a][0];
  }
  // W_i^T (.): row th_x += h_i row v ; row th_y -= h_i row u
#pragma unroll
  for (int b = 0; b < 6; ++b) {
    K[3][b] += hi * K[1][b];
    K[4][b] -= hi * K[0][b];
  }
  // each 3x3 block X -> R^T X R
#pragma unroll
  for (int bi = 0; bi < 2; ++bi)
#pragma unroll
    for (int bj = 0; bj < 2; ++bj) {
      double Y[3][3];
#pragma unroll
      for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int b = 0; b < 3; ++b)
          Y[a][b] = K[3 * bi + a][3 * bj + 0] * R[0][b] + K[3 * bi + a][3 * bj + 1] * R[1][b] +
                    K[3 * bi + a][3 * bj + 2] * R[2][b];
#pragma unroll
      for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int b = 0; b < 3; ++b)
          K[3 * bi + a][3 * bj + b] = R[0][a] * Y[0][b] + R[1][a] * Y[1][b] + R[2][a] * Y[2][b];
    }
}


}  // namespace shell
}  // namespace sso
