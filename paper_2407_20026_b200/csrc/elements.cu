// A1 — element stiffness kernels (sm_100a, fp64 CUDA cores), SURVEY.md §8(a) A1.
//
// Beam: 3D Euler-Bernoulli frame element (PAPER.md:75 element_K_bc_local, :112
// (E, G, Iy, Iz, J, A); reading c6).  Quad: flat 4-node MITC-4 shell
// (PAPER.md:44, 75-82 element_K_quad_local; reading c4: 2x2 Gauss, Dvorkin-Bathe
// tying, k_s = 5/6, coupled drilling gamma_d = alpha_d G, rigid-offset warping,
// intrinsic frame, kappa_x = kappa_y = 1).
//
// Mapping: one thread per (element, node-block (i, j)).  A quad has 16 node
// blocks of 6x6 (24x24 total); a CTA of 128 threads covers 8 quads.  Every
// thread recomputes the (cheap) element geometry, forms its 6x6 block of the
// local projected stiffness K_loc(i, j) over the 4 Gauss points, applies the
// warping map W and the rotation R (K_g = R6^T W_i^T K_loc W_j R6) and stages
// the block in shared memory; the CTA then writes its 128 consecutive staged
// blocks (36 KB) with fully coalesced stores.  Tensor cores are not used: the
// products are 6x6 and fp64 (BASELINE.json north_star).
#include <climits>

#include "shell_math.cuh"
#include "sso_internal.h"

namespace sso {

namespace {

using namespace sso::shell;

constexpr int QUADS_PER_CTA = 8;
constexpr int BEAMS_PER_CTA = 32;
constexpr int STAGE_PITCH = 37;  // padded 36 -> 37 doubles in smem (bank spread)

__global__ void __launch_bounds__(128) quad_element_kernel(
    int n_quads, const double* __restrict__ gx, const double* __restrict__ gy,
    const double* __restrict__ gz, const int32_t* __restrict__ conn,
    const double* __restrict__ gt, const double* __restrict__ gE,
    const double* __restrict__ gnu, double drill_alpha, double* __restrict__ stage,
    DevFlags* flags, BatchStrides bs) {
  __shared__ double sm[QUADS_PER_CTA * 16 * STAGE_PITCH];
  {  // design of a batch (blockIdx.y)
    const int bd = blockIdx.y;
    gx += bd * bs.node;
    gy += bd * bs.node;
    gz += bd * bs.node;
    gt += bd * bs.quad;
    stage += bd * bs.stage;
    flags += bd;
  }
  const int tid = threadIdx.x;
  const int le = tid >> 4, blk = tid & 15;
  const int bi = blk >> 2, bj = blk & 3;
  const int64_t q0 = (int64_t)blockIdx.x * QUADS_PER_CTA;
  const int64_t q = q0 + le;
  double K[6][6];
#pragma unroll
  for (int a = 0; a < 6; ++a)
#pragma unroll
    for (int b = 0; b < 6; ++b) K[a][b] = 0.0;

  if (q < n_quads) {
    double X[4][3];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      int n = __ldg(conn + 4 * q + k);
      X[k][0] = __ldg(gx + n);
      X[k][1] = __ldg(gy + n);
      X[k][2] = __ldg(gz + n);
    }
    const double t = __ldg(gt + q), E = __ldg(gE + q), nu = __ldg(gnu + q);
    // (a) frame
    double c[3], d13[3], d24[3], nrm[3], e1[3], e2[3], e3[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      c[a] = 0.25 * (X[0][a] + X[1][a] + X[2][a] + X[3][a]);
      d13[a] = X[2][a] - X[0][a];
      d24[a] = X[3][a] - X[1][a];
    }
    cross3(d13, d24, nrm);
    const double nn = sqrt(dot3(nrm, nrm));
    bool bad = !(nn > 0.0);
    const double inn = 1.0 / nn;
#pragma unroll
    for (int a = 0; a < 3; ++a) e3[a] = nrm[a] * inn;
    double d12[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) d12[a] = X[1][a] - X[0][a];
    const double p12 = dot3(d12, e3);
#pragma unroll
    for (int a = 0; a < 3; ++a) d12[a] -= p12 * e3[a];
    const double id = 1.0 / sqrt(dot3(d12, d12));
#pragma unroll
    for (int a = 0; a < 3; ++a) e1[a] = d12[a] * id;
    cross3(e3, e1, e2);
    double xl[4], yl[4];
    double hi = 0.0, hj = 0.0;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      double v[3] = {X[k][0] - c[0], X[k][1] - c[1], X[k][2] - c[2]};
      xl[k] = dot3(v, e1);
      yl[k] = dot3(v, e2);
      double hk = dot3(v, e3);
      if (k == bi) hi = hk;
      if (k == bj) hj = hk;
    }
    // material
    const double onu2 = 1.0 / (1.0 - nu * nu);
    const double Em = E * t * onu2;
    const double Eb = E * t * t * t * (1.0 / 12.0) * onu2;
    const double G = E / (2.0 * (1.0 + nu));
    const double ds = (5.0 / 6.0) * G * t;
    const double cs = 0.5 * (1.0 - nu);
    const double XIN[4] = {-1.0, 1.0, 1.0, -1.0};
    const double ETN[4] = {-1.0, -1.0, 1.0, 1.0};

    // (f) tying data for nodes bi and bj: xi-tying A (p=2,m=3) or C (p=1,m=0);
    // eta-tying D (p=2,m=1) or B (p=3,m=0); per node: coefficients (w, th_x, th_y)
    auto tying = [&](int k, bool xi_dir, double* g, int& side) {
      int p, m;
      if (xi_dir) {
        if (k == 2 || k == 3) { p = 2; m = 3; side = +1; } else { p = 1; m = 0; side = -1; }
      } else {
        if (k == 1 || k == 2) { p = 2; m = 1; side = +1; } else { p = 3; m = 0; side = -1; }
      }
      const double dx = 0.5 * (xl[p] - xl[m]);
      const double dy = 0.5 * (yl[p] - yl[m]);
      g[0] = (k == p) ? 0.5 : -0.5;  // w
      g[1] = -0.5 * dy;              // th_x  (beta_y = -th_x)
      g[2] = 0.5 * dx;               // th_y  (beta_x = th_y)
    };
    double gxi_i[3], geta_i[3], gxi_j[3], geta_j[3];
    int sxi_i, seta_i, sxi_j, seta_j;
    tying(bi, true, gxi_i, sxi_i);
    tying(bi, false, geta_i, seta_i);
    tying(bj, true, gxi_j, sxi_j);
    tying(bj, false, geta_j, seta_j);

    const double gpv = 0.57735026918962576451;  // 1/sqrt(3)
    const double GXI[4] = {-gpv, gpv, gpv, -gpv};
    const double GET[4] = {-gpv, -gpv, gpv, gpv};
    double area = 0.0;
#pragma unroll
    for (int g = 0; g < 4; ++g) {
      const double xi = GXI[g], eta = GET[g];
      double dxi[4], deta[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        dxi[k] = 0.25 * XIN[k] * (1.0 + ETN[k] * eta);
        deta[k] = 0.25 * ETN[k] * (1.0 + XIN[k] * xi);
      }
      double x_xi = 0, y_xi = 0, x_eta = 0, y_eta = 0;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        x_xi += dxi[k] * xl[k];
        y_xi += dxi[k] * yl[k];
        x_eta += deta[k] * xl[k];
        y_eta += deta[k] * yl[k];
      }
      const double detJ = x_xi * y_eta - y_xi * x_eta;
      bad |= !(detJ > 0.0);
      area += detJ;
      const double idet = 1.0 / detJ;
      const double j00 = y_eta * idet, j01 = -y_xi * idet, j10 = -x_eta * idet, j11 = x_xi * idet;
      const double Nxi = j00 * dxi[bi] + j01 * deta[bi], Nyi = j10 * dxi[bi] + j11 * deta[bi];
      const double Nxj = j00 * dxi[bj] + j01 * deta[bj], Nyj = j10 * dxi[bj] + j11 * deta[bj];
      // (d) membrane on (u, v)
      {
        const double s = Em * detJ;
        K[0][0] += s * (Nxi * Nxj + cs * Nyi * Nyj);
        K[0][1] += s * (nu * Nxi * Nyj + cs * Nyi * Nxj);
        K[1][0] += s * (nu * Nyi * Nxj + cs * Nxi * Nyj);
        K[1][1] += s * (Nyi * Nyj + cs * Nxi * Nxj);
      }
      // (e) bending on (th_x, th_y): B_b,k = [[0, Nx], [-Ny, 0], [-Nx, Ny]]
      {
        const double s = Eb * detJ;
        K[3][3] += s * (Nyi * Nyj + cs * Nxi * Nxj);
        K[3][4] += s * (-nu * Nyi * Nxj - cs * Nxi * Nyj);
        K[4][3] += s * (-nu * Nxi * Nyj - cs * Nyi * Nxj);
        K[4][4] += s * (Nxi * Nxj + cs * Nyi * Nyj);
      }
      // (f) MITC-4 shear on (w, th_x, th_y)
      {
        const double fxi_i = 0.5 * (1.0 + sxi_i * eta), feta_i = 0.5 * (1.0 + seta_i * xi);
        const double fxi_j = 0.5 * (1.0 + sxi_j * eta), feta_j = 0.5 * (1.0 + seta_j * xi);
        double bi0[3], bi1[3], bj0[3], bj1[3];
#pragma unroll
        for (int a = 0; a < 3; ++a) {
          const double gx_i = fxi_i * gxi_i[a], ge_i = feta_i * geta_i[a];
          const double gx_j = fxi_j * gxi_j[a], ge_j = feta_j * geta_j[a];
          bi0[a] = j00 * gx_i + j01 * ge_i;
          bi1[a] = j10 * gx_i + j11 * ge_i;
          bj0[a] = j00 * gx_j + j01 * ge_j;
          bj1[a] = j10 * gx_j + j11 * ge_j;
        }
        const double s = ds * detJ;
#pragma unroll
        for (int a = 0; a < 3; ++a)
#pragma unroll
          for (int b = 0; b < 3; ++b) K[2 + a][2 + b] += s * (bi0[a] * bj0[b] + bi1[a] * bj1[b]);
      }
    }
    // (g) drilling: omega_c = 1/2 (v,x - u,y) at the centre; b_k = e_thz_k - b_omega
    {
      double x_xi = 0, y_xi = 0, x_eta = 0, y_eta = 0;
      double dxi[4], deta[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        dxi[k] = 0.25 * XIN[k];
        deta[k] = 0.25 * ETN[k];
        x_xi += dxi[k] * xl[k];
        y_xi += dxi[k] * yl[k];
        x_eta += deta[k] * xl[k];
        y_eta += deta[k] * yl[k];
      }
      const double idet = 1.0 / (x_xi * y_eta - y_xi * x_eta);
      const double j00 = y_eta * idet, j01 = -y_xi * idet, j10 = -x_eta * idet, j11 = x_xi * idet;
      const double Nxi = j00 * dxi[bi] + j01 * deta[bi], Nyi = j10 * dxi[bi] + j11 * deta[bi];
      const double Nxj = j00 * dxi[bj] + j01 * deta[bj], Nyj = j10 * dxi[bj] + j11 * deta[bj];
      const double bwi[2] = {-0.5 * Nyi, 0.5 * Nxi};
      const double bwj[2] = {-0.5 * Nyj, 0.5 * Nxj};
      const double cd = drill_alpha * G * t * (area * 0.25);
#pragma unroll
      for (int a = 0; a < 2; ++a)
#pragma unroll
        for (int b = 0; b < 2; ++b) K[a][b] += 4.0 * cd * (bwi[a] * bwj[b]);
#pragma unroll
      for (int b = 0; b < 2; ++b) K[5][b] -= cd * bwj[b];
#pragma unroll
      for (int a = 0; a < 2; ++a) K[a][5] -= cd * bwi[a];
      if (bi == bj) K[5][5] += cd;
    }
    const double R[3][3] = {{e1[0], e1[1], e1[2]}, {e2[0], e2[1], e2[2]}, {e3[0], e3[1], e3[2]}};
    transform_block(K, R, hi, hj);
    if (bad && blk == 0) atomicMin(&flags->degenerate_elem, (int)q);
  }
  // stage in smem, then coalesced write of this CTA's consecutive blocks
  double* my = sm + tid * STAGE_PITCH;
#pragma unroll
  for (int a = 0; a < 6; ++a)
#pragma unroll
    for (int b = 0; b < 6; ++b) my[6 * a + b] = K[a][b];
  __syncthreads();
  const int64_t nq_here = min((int64_t)QUADS_PER_CTA, (int64_t)n_quads - q0);
  const int total = (int)(nq_here * 16 * 36);
  double* dst = stage + q0 * 16 * 36;
  for (int k = tid; k < total; k += blockDim.x) {
    const int b = k / 36, e = k - 36 * b;
    dst[k] = sm[b * STAGE_PITCH + e];
  }
}

// The distinct entries of the local 12x12 frame stiffness (reading C1), each formed once per
// element with the expressions (and so the rounding) of the entry table below.
struct BeamK {
  double ea, gj, z12, y12, z4, z2, y4, y2, z6, y6;
  __device__ BeamK(double EA, double GJ, double EIy, double EIz, double L) {
    const double L2 = L * L, L3 = L2 * L;
    ea = EA / L;
    gj = GJ / L;
    z12 = 12.0 * EIz / L3;
    y12 = 12.0 * EIy / L3;
    z4 = 4.0 * EIz / L;
    z2 = 2.0 * EIz / L;
    y4 = 4.0 * EIy / L;
    y2 = 2.0 * EIy / L;
    z6 = 6.0 * EIz / L2;
    y6 = 6.0 * EIy / L2;
  }
};

// Local 12x12 frame stiffness entry, local DOF (u, v, w, th_x, th_y, th_z).
__device__ __forceinline__ double beam_kloc(int r, int c, const BeamK& k) {
  if (r > c) { int tmp = r; r = c; c = tmp; }
  const int ra = r % 6, ca = c % 6;
  const bool same = (r / 6) == (c / 6);
  switch (ra * 6 + ca) {
    case 0 * 6 + 0: return same ? k.ea : -k.ea;
    case 3 * 6 + 3: return same ? k.gj : -k.gj;
    case 1 * 6 + 1: return same ? k.z12 : -k.z12;
    case 2 * 6 + 2: return same ? k.y12 : -k.y12;
    case 5 * 6 + 5: return same ? k.z4 : k.z2;
    case 4 * 6 + 4: return same ? k.y4 : k.y2;
    // v - th_z couplings: k(1,5) = k(1,11) = 6EIz/L^2 ; k(5,7) = k(7,11) = -6EIz/L^2
    case 1 * 6 + 5: return (r == 1) ? k.z6 : -k.z6;   // (1,5),(1,11) | (7,11)
    case 5 * 6 + 1: return -k.z6;                     // (5,7)
    // w - th_y couplings: k(2,4) = k(2,10) = -6EIy/L^2 ; k(4,8) = k(8,10) = +6EIy/L^2
    case 2 * 6 + 4: return (r == 2) ? -k.y6 : k.y6;   // (2,4),(2,10) | (8,10)
    case 4 * 6 + 2: return k.y6;                      // (4,8)
    default: return 0.0;
  }
}

__global__ void __launch_bounds__(128) beam_element_kernel(
    int n_beams, const double* __restrict__ gx, const double* __restrict__ gy,
    const double* __restrict__ gz, const int32_t* __restrict__ conn,
    const double* __restrict__ gA, const double* __restrict__ gIy,
    const double* __restrict__ gIz, const double* __restrict__ gJ,
    const double* __restrict__ gE, const double* __restrict__ gG, double* __restrict__ stage,
    DevFlags* flags, BatchStrides bs) {
  __shared__ double sm[BEAMS_PER_CTA * 4 * STAGE_PITCH];
  {  // design of a batch (blockIdx.y)
    const int bd = blockIdx.y;
    gx += bd * bs.node;
    gy += bd * bs.node;
    gz += bd * bs.node;
    stage += bd * bs.stage;
    flags += bd;
  }
  const int tid = threadIdx.x;
  const int le = tid >> 2, blk = tid & 3;
  const int bi = blk >> 1, bj = blk & 1;
  const int64_t e0 = (int64_t)blockIdx.x * BEAMS_PER_CTA;
  const int64_t e = e0 + le;
  double K[6][6];
#pragma unroll
  for (int a = 0; a < 6; ++a)
#pragma unroll
    for (int b = 0; b < 6; ++b) K[a][b] = 0.0;
  if (e < n_beams) {
    const int ni = __ldg(conn + 2 * e), nj = __ldg(conn + 2 * e + 1);
    double d[3] = {__ldg(gx + nj) - __ldg(gx + ni), __ldg(gy + nj) - __ldg(gy + ni),
                   __ldg(gz + nj) - __ldg(gz + ni)};
    const double L = sqrt(dot3(d, d));
    if (!(L > 0.0)) {
      if (blk == 0) atomicMin(&flags->degenerate_elem, (int)e);
    } else {
      double ex[3] = {d[0] / L, d[1] / L, d[2] / L};
      double a[3] = {0.0, 0.0, 1.0};
      if (fabs(ex[2]) > 0.99999999999950000) {  // cos(1e-6)
        a[0] = 1.0;
        a[2] = 0.0;
      }
      const double ax = dot3(a, ex);
      double w[3] = {a[0] - ax * ex[0], a[1] - ax * ex[1], a[2] - ax * ex[2]};
      const double iw = 1.0 / sqrt(dot3(w, w));
      double ez[3] = {w[0] * iw, w[1] * iw, w[2] * iw};
      double ey[3];
      cross3(ez, ex, ey);
      const double E = __ldg(gE + e);
      const double EA = E * __ldg(gA + e), GJ = __ldg(gG + e) * __ldg(gJ + e);
      const double EIy = E * __ldg(gIy + e), EIz = E * __ldg(gIz + e);
      const BeamK kk(EA, GJ, EIy, EIz, L);
#pragma unroll
      for (int a2 = 0; a2 < 6; ++a2)
#pragma unroll
        for (int b2 = 0; b2 < 6; ++b2) K[a2][b2] = beam_kloc(6 * bi + a2, 6 * bj + b2, kk);
      const double R[3][3] = {{ex[0], ex[1], ex[2]}, {ey[0], ey[1], ey[2]}, {ez[0], ez[1], ez[2]}};
      transform_block(K, R, 0.0, 0.0);
    }
  }
  double* my = sm + tid * STAGE_PITCH;
#pragma unroll
  for (int a = 0; a < 6; ++a)
#pragma unroll
    for (int b = 0; b < 6; ++b) my[6 * a + b] = K[a][b];
  __syncthreads();
  const int64_t nb_here = min((int64_t)BEAMS_PER_CTA, (int64_t)n_beams - e0);
  const int total = (int)(nb_here * 4 * 36);
  double* dst = stage + e0 * 4 * 36;
  for (int k = tid; k < total; k += blockDim.x) {
    const int b = k / 36, ee = k - 36 * b;
    dst[k] = sm[b * STAGE_PITCH + ee];
  }
}

}  // namespace

void launch_quad_elements(cudaStream_t s, int n_quads, const double* x, const double* y,
                          const double* z, const int32_t* conn, const double* t,
                          const double* E, const double* nu, double drill_alpha,
                          double* stage, DevFlags* flags, const BatchStrides& bs) {
  if (n_quads <= 0) return;
  const dim3 grid((n_quads + QUADS_PER_CTA - 1) / QUADS_PER_CTA, bs.B);
  quad_element_kernel<<<grid, 128, 0, s>>>(n_quads, x, y, z, conn, t, E, nu, drill_alpha, stage,
                                           flags, bs);
  SSO_POST_LAUNCH("quad_element_kernel");
}

void launch_beam_elements(cudaStream_t s, int n_beams, const double* x, const double* y,
                          const double* z, const int32_t* conn, const double* A,
                          const double* Iy, const double* Iz, const double* J,
                          const double* E, const double* G, double* stage, DevFlags* flags,
                          const BatchStrides& bs) {
  if (n_beams <= 0) return;
  const dim3 grid((n_beams + BEAMS_PER_CTA - 1) / BEAMS_PER_CTA, bs.B);
  beam_element_kernel<<<grid, 128, 0, s>>>(n_beams, x, y, z, conn, A, Iy, Iz, J, E, G, stage,
                                           flags, bs);
  SSO_POST_LAUNCH("beam_element_kernel");
}

}  // namespace sso
