// A1 + A2 fused for quad-shell meshes (sm_100a): element stiffness and the
// atomic-free assembly in ONE pass, with no staged element matrices.
//
// Same mathematics as elements.cu (reading c4) and
// assemble.cu (ascending-element sums, elimination supports, Jacobi diagonal);
// the difference is the data flow.  A CTA owns NPC consecutive nodes.  For
// each node, each incident quad and each column block j, one thread forms the
// 6x6 block (i, j) of that quad (i = the node's local index): exactly the
// blocks of the node's six CSR rows, so no block is computed twice.  The
// per-(node, element) geometry (frame, warp offsets, Gauss-point shape
// derivatives, Jacobians, tying data, material) is computed once into shared
// memory and read by the node's 4 column-block threads.  Blocks are added to
// the node's CSR run held in shared memory in ascending element order (the
// order of the staged path), then supports and dinv are applied and the run is
// written once, coalesced.  HBM traffic is the CSR values written once plus the
// (L2-resident) coordinates: the staged path's 2 x 36 x 16 x 8 B per quad of
// element-matrix staging disappears.  Latency: each (node, incident quad) reads one
// 32-byte incidence record {quad, local index, its 4 nodes, its 4 block ranks} built on the
// host, so the load chain is record -> coordinates (was node -> incidence -> quad ->
// connectivity -> coordinates, + block rank), and the column blocks' fixed masks are staged
// in shared memory at the start (C3b: 0.419 -> 0.374 ms).
#include <climits>

#include "shell_math.cuh"
#include "sso_internal.h"

namespace sso {

namespace {

using namespace sso::shell;

constexpr int NPC = 8;         // nodes per CTA (16 threads each)
constexpr int MAXDEG = 10;     // node-graph degree handled by the fused path (grids: 9)
constexpr int GS = 89;         // doubles per geometry record (odd: conflict-free 8-record reads)
enum {
  G_R = 0, G_H = 9, G_DET = 13, G_NX = 17, G_NY = 33, G_JI = 49, G_TX = 65, G_TY = 69,
  G_NX0 = 73, G_NY0 = 77, G_EM = 81, G_EB = 82, G_DS = 83, G_CS = 84, G_NU = 85, G_CD = 86
};

// tying points A (p=2, m=3), C (p=1, m=0), D (p=2, m=1), B (p=3, m=0)
__device__ __forceinline__ void node_tying(int k, bool xi_dir, const double* G, double* g, int& side) {
  int t, p;
  if (xi_dir) {
    if (k == 2 || k == 3) { t = 0; p = 2; side = +1; } else { t = 1; p = 1; side = -1; }
  } else {
    if (k == 1 || k == 2) { t = 2; p = 2; side = +1; } else { t = 3; p = 3; side = -1; }
  }
  g[0] = (k == p) ? 0.5 : -0.5;   // w
  g[1] = -0.5 * G[G_TY + t];      // th_x (beta_y = -th_x)
  g[2] = 0.5 * G[G_TX + t];       // th_y (beta_x = th_y)
}

__global__ void __launch_bounds__(128, 4) quad_assemble_fused_kernel(
    int n_own, int inc_pad, const int64_t* __restrict__ node_ptr, const int32_t* __restrict__ node_col,
    const int32_t* __restrict__ inc_rec, const double* __restrict__ gx, const double* __restrict__ gy,
    const double* __restrict__ gz, const double* __restrict__ gt,
    const double* __restrict__ gE, const double* __restrict__ gnu, double drill_alpha,
    const uint8_t* __restrict__ fixed_mask, double* __restrict__ vals, double* __restrict__ dinv,
    DevFlags* flags, BatchStrides bs, int cm) {
  __shared__ double geo[NPC * 4 * GS];
  __shared__ double buf[NPC * 36 * MAXDEG];
  __shared__ uint16_t ccol[NPC][MAXDEG];  // per column block: fixed mask of its node | self << 8
  {  // design of a batch (blockIdx.y)
    const int bd = blockIdx.y;
    gx += bd * bs.node;
    gy += bd * bs.node;
    gz += bd * bs.node;
    gt += bd * bs.quad;
    vals += bd * bs.nnz;
    dinv += bd * bs.dof;
    flags += bd;
  }
  const int tid = threadIdx.x;
  const int ns = tid >> 4;            // node slot in the CTA
  const int k = (tid >> 2) & 3;       // incident element within a group of 4
  const int j = tid & 3;              // column block (element-local node)
  const int t16 = tid & 15;
  const int64_t n = (int64_t)blockIdx.x * NPC + ns;
  const bool node_ok = n < n_own;
  int64_t b0 = 0;
  int deg = 0;
  if (node_ok) {
    b0 = node_ptr[n];
    deg = (int)(node_ptr[n + 1] - b0);
  }
  const int rowlen = 6 * deg;
  double* nbuf = buf + ns * 36 * MAXDEG;
  for (int v = t16; v < 36 * deg; v += 16) nbuf[v] = 0.0;
  if (t16 < deg) {  // off the write phase's critical path (read after the group loop's barrier)
    const int m = node_col[b0 + t16];
    ccol[ns][t16] = (uint16_t)(fixed_mask[m] | (m == n ? 256 : 0));
  }

  for (int grp = 0; grp * 4 < inc_pad; ++grp) {
    const int kk = grp * 4 + k;
    // incidence record {quad, local index, its 4 nodes, 4 int8 block ranks}: one load level
    int4 r0 = make_int4(-1, 0, 0, 0), r1 = make_int4(0, 0, 0, 0);
    if (node_ok) {
      const int4* rp = reinterpret_cast<const int4*>(inc_rec + 8 * (n * inc_pad + kk));
      r0 = __ldg(rp);
      r1 = __ldg(rp + 1);
    }
    const bool has = r0.x >= 0;
    const int64_t q = has ? r0.x : 0;
    const int il = r0.y;
    const int cn[4] = {r0.z, r0.w, r1.x, r1.y};
    double* G = geo + (ns * 4 + k) * GS;
    // ---- phase 1: geometry of (node, element) once ------------------------
    if (has && j == 0) {
      double X[4][3];
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const int m = cn[c];
        X[c][0] = __ldg(gx + m);
        X[c][1] = __ldg(gy + m);
        X[c][2] = __ldg(gz + m);
      }
      const double t = __ldg(gt + q), E = __ldg(gE + q), nu = __ldg(gnu + q);
      double c0[3], d13[3], d24[3], nrm[3], e1[3], e2[3], e3[3], d12[3];
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        c0[a] = 0.25 * (X[0][a] + X[1][a] + X[2][a] + X[3][a]);
        d13[a] = X[2][a] - X[0][a];
        d24[a] = X[3][a] - X[1][a];
        d12[a] = X[1][a] - X[0][a];
      }
      cross3(d13, d24, nrm);
      const double nn = sqrt(dot3(nrm, nrm));
      bool bad = !(nn > 0.0);
      const double inn = 1.0 / nn;
#pragma unroll
      for (int a = 0; a < 3; ++a) e3[a] = nrm[a] * inn;
      const double p12 = dot3(d12, e3);
#pragma unroll
      for (int a = 0; a < 3; ++a) d12[a] -= p12 * e3[a];
      const double id = 1.0 / sqrt(dot3(d12, d12));
#pragma unroll
      for (int a = 0; a < 3; ++a) e1[a] = d12[a] * id;
      cross3(e3, e1, e2);
      double xl[4], yl[4];
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        double v[3] = {X[c][0] - c0[0], X[c][1] - c0[1], X[c][2] - c0[2]};
        xl[c] = dot3(v, e1);
        yl[c] = dot3(v, e2);
        G[G_H + c] = dot3(v, e3);
      }
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        G[G_R + a] = e1[a];
        G[G_R + 3 + a] = e2[a];
        G[G_R + 6 + a] = e3[a];
      }
      const double XIN[4] = {-1.0, 1.0, 1.0, -1.0};
      const double ETN[4] = {-1.0, -1.0, 1.0, 1.0};
      const double gpv = 0.57735026918962576451;
      const double GXI[4] = {-gpv, gpv, gpv, -gpv};
      const double GET[4] = {-gpv, -gpv, gpv, gpv};
      double area = 0.0;
#pragma unroll
      for (int g = 0; g < 4; ++g) {
        const double xi = GXI[g], eta = GET[g];
        double dxi[4], deta[4];
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          dxi[c] = 0.25 * XIN[c] * (1.0 + ETN[c] * eta);
          deta[c] = 0.25 * ETN[c] * (1.0 + XIN[c] * xi);
        }
        double x_xi = 0, y_xi = 0, x_eta = 0, y_eta = 0;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          x_xi += dxi[c] * xl[c];
          y_xi += dxi[c] * yl[c];
          x_eta += deta[c] * xl[c];
          y_eta += deta[c] * yl[c];
        }
        const double detJ = x_xi * y_eta - y_xi * x_eta;
        bad |= !(detJ > 0.0);
        area += detJ;
        const double idet = 1.0 / detJ;
        const double j00 = y_eta * idet, j01 = -y_xi * idet, j10 = -x_eta * idet, j11 = x_xi * idet;
        G[G_DET + g] = detJ;
        G[G_JI + 4 * g + 0] = j00;
        G[G_JI + 4 * g + 1] = j01;
        G[G_JI + 4 * g + 2] = j10;
        G[G_JI + 4 * g + 3] = j11;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          G[G_NX + 4 * g + c] = j00 * dxi[c] + j01 * deta[c];
          G[G_NY + 4 * g + c] = j10 * dxi[c] + j11 * deta[c];
        }
      }
      {  // centre (drilling)
        double x_xi = 0, y_xi = 0, x_eta = 0, y_eta = 0;
        double dxi[4], deta[4];
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          dxi[c] = 0.25 * XIN[c];
          deta[c] = 0.25 * ETN[c];
          x_xi += dxi[c] * xl[c];
          y_xi += dxi[c] * yl[c];
          x_eta += deta[c] * xl[c];
          y_eta += deta[c] * yl[c];
        }
        const double idet = 1.0 / (x_xi * y_eta - y_xi * x_eta);
        const double j00 = y_eta * idet, j01 = -y_xi * idet, j10 = -x_eta * idet, j11 = x_xi * idet;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          G[G_NX0 + c] = j00 * dxi[c] + j01 * deta[c];
          G[G_NY0 + c] = j10 * dxi[c] + j11 * deta[c];
        }
      }
      // tying points A, C, D, B: half-edge vectors 1/2 (x_p - x_m)
      const int TP[4] = {2, 1, 2, 3}, TM[4] = {3, 0, 1, 0};
#pragma unroll
      for (int tpt = 0; tpt < 4; ++tpt) {
        G[G_TX + tpt] = 0.5 * (xl[TP[tpt]] - xl[TM[tpt]]);
        G[G_TY + tpt] = 0.5 * (yl[TP[tpt]] - yl[TM[tpt]]);
      }
      const double onu2 = 1.0 / (1.0 - nu * nu);
      const double Gm = E / (2.0 * (1.0 + nu));
      G[G_EM] = E * t * onu2;
      G[G_EB] = E * t * t * t * (1.0 / 12.0) * onu2;
      G[G_DS] = (5.0 / 6.0) * Gm * t;
      G[G_CS] = 0.5 * (1.0 - nu);
      G[G_NU] = nu;
      G[G_CD] = drill_alpha * Gm * t * (area * 0.25);
      if (bad) atomicMin(&flags->degenerate_elem, (int)q);
    }
    __syncthreads();
    // ---- phase 2: block (il, j) of element q --------------------------------
    double K[6][6];
#pragma unroll
    for (int a = 0; a < 6; ++a)
#pragma unroll
      for (int b = 0; b < 6; ++b) K[a][b] = 0.0;
    // symmetric storage keeps only blocks (n, m >= n): rank < 0 marks a skipped block
    const int rank = has ? (int)(int8_t)((r1.z >> (8 * j)) & 255) : -1;
    const bool blk = has && rank >= 0;
    if (blk) {
      const int bi = il, bj = j;
      const double Em = G[G_EM], Eb = G[G_EB], ds = G[G_DS], cs = G[G_CS], nu = G[G_NU];
      double gxi_i[3], geta_i[3], gxi_j[3], geta_j[3];
      int sxi_i, seta_i, sxi_j, seta_j;
      node_tying(bi, true, G, gxi_i, sxi_i);
      node_tying(bi, false, G, geta_i, seta_i);
      node_tying(bj, true, G, gxi_j, sxi_j);
      node_tying(bj, false, G, geta_j, seta_j);
      const double gpv = 0.57735026918962576451;
      const double GXI[4] = {-gpv, gpv, gpv, -gpv};
      const double GET[4] = {-gpv, -gpv, gpv, gpv};
#pragma unroll
      for (int g = 0; g < 4; ++g) {
        const double xi = GXI[g], eta = GET[g];
        const double detJ = G[G_DET + g];
        const double Nxi = G[G_NX + 4 * g + bi], Nyi = G[G_NY + 4 * g + bi];
        const double Nxj = G[G_NX + 4 * g + bj], Nyj = G[G_NY + 4 * g + bj];
        {
          const double s = Em * detJ;
          K[0][0] += s * (Nxi * Nxj + cs * Nyi * Nyj);
          K[0][1] += s * (nu * Nxi * Nyj + cs * Nyi * Nxj);
          K[1][0] += s * (nu * Nyi * Nxj + cs * Nxi * Nyj);
          K[1][1] += s * (Nyi * Nyj + cs * Nxi * Nxj);
        }
        {
          const double s = Eb * detJ;
          K[3][3] += s * (Nyi * Nyj + cs * Nxi * Nxj);
          K[3][4] += s * (-nu * Nyi * Nxj - cs * Nxi * Nyj);
          K[4][3] += s * (-nu * Nxi * Nyj - cs * Nyi * Nxj);
          K[4][4] += s * (Nxi * Nxj + cs * Nyi * Nyj);
        }
        {
          const double j00 = G[G_JI + 4 * g], j01 = G[G_JI + 4 * g + 1];
          const double j10 = G[G_JI + 4 * g + 2], j11 = G[G_JI + 4 * g + 3];
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
      {
        const double Nxi = G[G_NX0 + bi], Nyi = G[G_NY0 + bi];
        const double Nxj = G[G_NX0 + bj], Nyj = G[G_NY0 + bj];
        const double bwi[2] = {-0.5 * Nyi, 0.5 * Nxi};
        const double bwj[2] = {-0.5 * Nyj, 0.5 * Nxj};
        const double cd = G[G_CD];
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
      const double R[3][3] = {{G[G_R + 0], G[G_R + 1], G[G_R + 2]},
                              {G[G_R + 3], G[G_R + 4], G[G_R + 5]},
                              {G[G_R + 6], G[G_R + 7], G[G_R + 8]}};
      transform_block(K, R, G[G_H + bi], G[G_H + bj]);
    }
    // ---- ordered accumulation into the node's CSR run (ascending element) ----
#pragma unroll
    for (int kk2 = 0; kk2 < 4; ++kk2) {
      if (blk && k == kk2) {
#pragma unroll
        for (int a = 0; a < 6; ++a)
#pragma unroll
          for (int b = 0; b < 6; ++b) nbuf[a * rowlen + 6 * rank + b] += K[a][b];
      }
      __syncwarp();
    }
    __syncthreads();  // geometry records are reused by the next group
  }
  // ---- supports (elimination), Jacobi diagonal, one coalesced write ----------
  if (node_ok) {
    const uint8_t mrow = fixed_mask[n];
    // run layout: row-major (a, rem) runs of 36 deg values, or (cm) one PULL_BLOCK record per
    // block (2x2 sub-blocks, rec_off); v walks the values block by block
    double* out = vals + (cm ? PULL_BLOCK : 36) * b0;
    for (int v = t16; v < 36 * deg; v += 16) {
      const int a = cm ? v % 6 : v / rowlen;
      const int rem = cm ? v / 6 : v - a * rowlen;
      const int kb = rem / 6;
      const int b = rem - 6 * kb;
      const int dst = cm ? PULL_BLOCK * kb + rec_off(a, b) : v;
      const int cc = ccol[ns][kb];
      double s = nbuf[a * rowlen + rem];
      const bool diag = (cc >> 8) && (a == b);
      const bool rfix = (mrow >> a) & 1;
      const bool cfix = (cc >> b) & 1;
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

int fused_max_degree() { return MAXDEG; }

void launch_quad_assemble_fused(cudaStream_t s, int n_own, int inc_pad, const int64_t* node_ptr,
                                const int32_t* node_col, const int32_t* inc_rec, const double* x,
                                const double* y, const double* z, const double* t, const double* E,
                                const double* nu, double drill_alpha, const uint8_t* fixed_mask,
                                double* vals, double* dinv, DevFlags* flags, const BatchStrides& bs,
                                int cm) {
  if (n_own <= 0) return;
  const dim3 grid((n_own + NPC - 1) / NPC, bs.B);
  quad_assemble_fused_kernel<<<grid, 128, 0, s>>>(n_own, inc_pad, node_ptr, node_col, inc_rec, x, y, z, t, E,
                                                  nu, drill_alpha,
                                                  fixed_mask, vals, dinv, flags, bs, cm);
  SSO_POST_LAUNCH("quad_assemble_fused_kernel");
}

}  // namespace sso
