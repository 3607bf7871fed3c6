// A4 — compliance and element-wise adjoint gradient (sm_100a), SURVEY.md §8(a) A4.
//
// PAPER.md:212-221 (Eq. 5-6).  For g = s f^T u with f fixed (reading c3) and K
// symmetric, the adjoint state is lambda = s u and Eq. 6 reduces to
//     dC/dp = -s sum_e u_e^T (dK_e/dp) u_e = -s sum_e d/dp [ u_e^T K_e(p) u_e ] |_{u fixed}
// (s = 1 compliance, s = 1/2 strain energy, reading c2).
//
// The element strain energy u_e^T K_e u_e is evaluated directly from strains
// (membrane, bending, MITC-4 shear, drilling; reading c4 / C2) with
// forward-mode dual numbers, one thread per (element, design parameter):
// 12 node coordinates + thickness for a quad (13 of 16 lanes), 6 coordinates
// for a beam (6 of 8 lanes).  Per-element-node coordinate partials are
// written to slots (2e+i beams, 2Eb+4q+i quads) and summed per node over the
// node->element incidence in ascending element order (node_reduce_kernel):
// deterministic, atomic-free.
#include "sso_internal.h"

namespace sso {

namespace {

struct Dual {
  double v, d;
  __device__ Dual() : v(0.0), d(0.0) {}
  __device__ Dual(double a) : v(a), d(0.0) {}
  __device__ Dual(double a, double b) : v(a), d(b) {}
};
__device__ __forceinline__ Dual operator+(Dual a, Dual b) { return Dual(a.v + b.v, a.d + b.d); }
__device__ __forceinline__ Dual operator-(Dual a, Dual b) { return Dual(a.v - b.v, a.d - b.d); }
__device__ __forceinline__ Dual operator-(Dual a) { return Dual(-a.v, -a.d); }
__device__ __forceinline__ Dual operator*(Dual a, Dual b) {
  return Dual(a.v * b.v, a.d * b.v + a.v * b.d);
}
__device__ __forceinline__ Dual operator*(double a, Dual b) { return Dual(a * b.v, a * b.d); }
__device__ __forceinline__ Dual operator*(Dual a, double b) { return Dual(a.v * b, a.d * b); }
__device__ __forceinline__ Dual operator/(Dual a, Dual b) {
  const double iv = 1.0 / b.v;
  const double q = a.v * iv;
  return Dual(q, (a.d - q * b.d) * iv);
}
__device__ __forceinline__ Dual operator/(double a, Dual b) { return Dual(a) / b; }
__device__ __forceinline__ Dual& operator+=(Dual& a, Dual b) { a.v += b.v; a.d += b.d; return a; }
__device__ __forceinline__ Dual& operator-=(Dual& a, Dual b) { a.v -= b.v; a.d -= b.d; return a; }
__device__ __forceinline__ Dual dsqrt(Dual a) {
  const double s = sqrt(a.v);
  return Dual(s, a.d * 0.5 / s);
}

template <class T>
__device__ __forceinline__ T dot3(const T* a, const T* b) {
  return a[0] * b[0] + a[1] * b[1] + a[2] * b[2];
}
template <class T>
__device__ __forceinline__ void cross3(const T* a, const T* b, T* c) {
  c[0] = a[1] * b[2] - a[2] * b[1];
  c[1] = a[2] * b[0] - a[0] * b[2];
  c[2] = a[0] * b[1] - a[1] * b[0];
}

// u_e^T K_e u_e of a flat MITC-4 quad (reading C2 (a)-(h)); X [4][3], u [24] global.
// BI: the bilinear form v_e^T K_e u_e instead (the general adjoint -lambda^T dK/dp u, PAPER.md
// Eq. 6): every strain measure is formed for both states and each quadratic product s_i s_j
// of the energy becomes s_i(v) s_j(u) (symmetrised for the cross terms), one pass, no
// polarization.
template <bool BI>
__device__ Dual quad_energy(const Dual (&X)[4][3], Dual t, double E, double nu, double alpha_d,
                            const double (&u)[24], const double (&vb)[24]) {
  Dual c[3], d13[3], d24[3], nv[3], e1[3], e2[3], e3[3], d12[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    c[a] = 0.25 * (X[0][a] + X[1][a] + X[2][a] + X[3][a]);
    d13[a] = X[2][a] - X[0][a];
    d24[a] = X[3][a] - X[1][a];
    d12[a] = X[1][a] - X[0][a];
  }
  cross3(d13, d24, nv);
  const Dual inn = 1.0 / dsqrt(dot3(nv, nv));
#pragma unroll
  for (int a = 0; a < 3; ++a) e3[a] = nv[a] * inn;
  const Dual p12 = dot3(d12, e3);
#pragma unroll
  for (int a = 0; a < 3; ++a) d12[a] -= p12 * e3[a];
  const Dual id = 1.0 / dsqrt(dot3(d12, d12));
#pragma unroll
  for (int a = 0; a < 3; ++a) e1[a] = d12[a] * id;
  cross3(e3, e1, e2);
  // local coordinates and projected local displacements (state a = u; state b = vb when BI)
  Dual xl[4], yl[4], uP[4], vP[4], w[4], tx[4], ty[4], tz[4];
  Dual uPb[4], vPb[4], wb[4], txb[4], tyb[4], tzb[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    Dual v[3] = {X[k][0] - c[0], X[k][1] - c[1], X[k][2] - c[2]};
    xl[k] = dot3(v, e1);
    yl[k] = dot3(v, e2);
    const Dual h = dot3(v, e3);
    auto project = [&](const double (&uu)[24], Dual& oU, Dual& oV, Dual& oW, Dual& oX, Dual& oY, Dual& oZ) {
      const double* ut = &uu[6 * k];
      const double* ur = &uu[6 * k + 3];
      const Dual t0 = e1[0] * ut[0] + e1[1] * ut[1] + e1[2] * ut[2];
      const Dual t1 = e2[0] * ut[0] + e2[1] * ut[1] + e2[2] * ut[2];
      const Dual t2 = e3[0] * ut[0] + e3[1] * ut[1] + e3[2] * ut[2];
      const Dual r0 = e1[0] * ur[0] + e1[1] * ur[1] + e1[2] * ur[2];
      const Dual r1 = e2[0] * ur[0] + e2[1] * ur[1] + e2[2] * ur[2];
      const Dual r2 = e3[0] * ur[0] + e3[1] * ur[1] + e3[2] * ur[2];
      oU = t0 - h * r1;   // u_P = u - h th_y
      oV = t1 + h * r0;   // v_P = v + h th_x
      oW = t2;
      oX = r0;
      oY = r1;
      oZ = r2;
    };
    project(u, uP[k], vP[k], w[k], tx[k], ty[k], tz[k]);
    if (BI) project(vb, uPb[k], vPb[k], wb[k], txb[k], tyb[k], tzb[k]);
  }
  const double onu2 = 1.0 / (1.0 - nu * nu);
  const Dual Em = (E * onu2) * t;
  const Dual Eb = (E * onu2 / 12.0) * (t * t * t);
  const double G = E / (2.0 * (1.0 + nu));
  const Dual ds = ((5.0 / 6.0) * G) * t;
  const double cs = 0.5 * (1.0 - nu);
  // MITC-4 tying strains: gamma = 1/2 (w_p - w_m) + 1/2 (beta_p + beta_m) . 1/2 (x_p - x_m)
  auto tie = [&](int p, int m, const Dual* W, const Dual* TX, const Dual* TY) -> Dual {
    const Dual dx = 0.5 * (xl[p] - xl[m]);
    const Dual dy = 0.5 * (yl[p] - yl[m]);
    return 0.5 * (W[p] - W[m]) + 0.5 * ((TY[p] + TY[m]) * dx - (TX[p] + TX[m]) * dy);
  };
  const Dual gA = tie(2, 3, w, tx, ty), gC = tie(1, 0, w, tx, ty), gD = tie(2, 1, w, tx, ty),
             gB = tie(3, 0, w, tx, ty);
  Dual gAb, gCb, gDb, gBb;
  if (BI) {
    gAb = tie(2, 3, wb, txb, tyb);
    gCb = tie(1, 0, wb, txb, tyb);
    gDb = tie(2, 1, wb, txb, tyb);
    gBb = tie(3, 0, wb, txb, tyb);
  }
  const double XIN[4] = {-1.0, 1.0, 1.0, -1.0};
  const double ETN[4] = {-1.0, -1.0, 1.0, 1.0};
  const double gpv = 0.57735026918962576451;
  const double GXI[4] = {-gpv, gpv, gpv, -gpv};
  const double GET[4] = {-gpv, -gpv, gpv, gpv};
  Dual energy(0.0), area(0.0);
#pragma unroll
  for (int g = 0; g < 4; ++g) {
    const double xi = GXI[g], eta = GET[g];
    double dxi[4], deta[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      dxi[k] = 0.25 * XIN[k] * (1.0 + ETN[k] * eta);
      deta[k] = 0.25 * ETN[k] * (1.0 + XIN[k] * xi);
    }
    Dual x_xi(0.0), y_xi(0.0), x_eta(0.0), y_eta(0.0);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      x_xi += dxi[k] * xl[k];
      y_xi += dxi[k] * yl[k];
      x_eta += deta[k] * xl[k];
      y_eta += deta[k] * yl[k];
    }
    const Dual detJ = x_xi * y_eta - y_xi * x_eta;
    area += detJ;
    const Dual idet = 1.0 / detJ;
    const Dual j00 = y_eta * idet, j01 = -(y_xi * idet), j10 = -(x_eta * idet), j11 = x_xi * idet;
    Dual e0(0.0), e1m(0.0), e2m(0.0), k0(0.0), k1(0.0), k2(0.0);
    Dual e0b(0.0), e1mb(0.0), e2mb(0.0), k0b(0.0), k1b(0.0), k2b(0.0);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const Dual Nx = j00 * dxi[k] + j01 * deta[k];
      const Dual Ny = j10 * dxi[k] + j11 * deta[k];
      e0 += Nx * uP[k];
      e1m += Ny * vP[k];
      e2m += Ny * uP[k] + Nx * vP[k];
      k0 += Nx * ty[k];
      k1 -= Ny * tx[k];
      k2 += Ny * ty[k] - Nx * tx[k];
      if (BI) {
        e0b += Nx * uPb[k];
        e1mb += Ny * vPb[k];
        e2mb += Ny * uPb[k] + Nx * vPb[k];
        k0b += Nx * tyb[k];
        k1b -= Ny * txb[k];
        k2b += Ny * tyb[k] - Nx * txb[k];
      }
    }
    const Dual gxi = 0.5 * (1.0 + eta) * gA + 0.5 * (1.0 - eta) * gC;
    const Dual geta = 0.5 * (1.0 + xi) * gD + 0.5 * (1.0 - xi) * gB;
    const Dual gxz = j00 * gxi + j01 * geta;
    const Dual gyz = j10 * gxi + j11 * geta;
    if (!BI) {
      const Dual em = e0 * e0 + e1m * e1m + 2.0 * nu * (e0 * e1m) + cs * (e2m * e2m);
      const Dual eb = k0 * k0 + k1 * k1 + 2.0 * nu * (k0 * k1) + cs * (k2 * k2);
      energy += detJ * (Em * em + Eb * eb + ds * (gxz * gxz + gyz * gyz));
    } else {
      const Dual gxib = 0.5 * (1.0 + eta) * gAb + 0.5 * (1.0 - eta) * gCb;
      const Dual getab = 0.5 * (1.0 + xi) * gDb + 0.5 * (1.0 - xi) * gBb;
      const Dual gxzb = j00 * gxib + j01 * getab;
      const Dual gyzb = j10 * gxib + j11 * getab;
      const Dual em = e0b * e0 + e1mb * e1m + nu * (e0b * e1m + e1mb * e0) + cs * (e2mb * e2m);
      const Dual eb = k0b * k0 + k1b * k1 + nu * (k0b * k1 + k1b * k0) + cs * (k2b * k2);
      energy += detJ * (Em * em + Eb * eb + ds * (gxzb * gxz + gyzb * gyz));
    }
  }
  // drilling: alpha_d G t (A_e / 4) sum_k (th_z_k - omega_c)^2, omega_c = 1/2 (v,x - u,y) at centre
  {
    Dual x_xi(0.0), y_xi(0.0), x_eta(0.0), y_eta(0.0);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      x_xi += (0.25 * XIN[k]) * xl[k];
      y_xi += (0.25 * XIN[k]) * yl[k];
      x_eta += (0.25 * ETN[k]) * xl[k];
      y_eta += (0.25 * ETN[k]) * yl[k];
    }
    const Dual idet = 1.0 / (x_xi * y_eta - y_xi * x_eta);
    const Dual j00 = y_eta * idet, j01 = -(y_xi * idet), j10 = -(x_eta * idet), j11 = x_xi * idet;
    Dual om(0.0), omb(0.0);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const Dual Nx = j00 * (0.25 * XIN[k]) + j01 * (0.25 * ETN[k]);
      const Dual Ny = j10 * (0.25 * XIN[k]) + j11 * (0.25 * ETN[k]);
      om += 0.5 * (Nx * vP[k] - Ny * uP[k]);
      if (BI) omb += 0.5 * (Nx * vPb[k] - Ny * uPb[k]);
    }
    Dual sq(0.0);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const Dual dd = tz[k] - om;
      if (BI) sq += (tzb[k] - omb) * dd;
      else sq += dd * dd;
    }
    energy += ((alpha_d * G) * t) * (0.25 * area) * sq;
  }
  return energy;
}

template <bool BI>
__global__ void __launch_bounds__(128) quad_grad_kernel(
    int n_beams, int n_quads, const double* __restrict__ gx, const double* __restrict__ gy,
    const double* __restrict__ gz, const int32_t* __restrict__ conn,
    const double* __restrict__ gt, const double* __restrict__ gE,
    const double* __restrict__ gnu, double drill_alpha, const double* __restrict__ u,
    const double* __restrict__ vb, double scale, double* __restrict__ slot_partial, double* __restrict__ dC_dt,
    double* __restrict__ dC_dE, int n_elems, BatchStrides bs) {
  {  // design of a batch (blockIdx.y)
    const int bd = blockIdx.y;
    gx += bd * bs.node;
    gy += bd * bs.node;
    gz += bd * bs.node;
    gt += bd * bs.quad;
    u += bd * bs.dof;
    if (BI) vb += bd * bs.dof;
    slot_partial += bd * bs.slot;
    dC_dt += bd * bs.quad;
    if (dC_dE) dC_dE += bd * (int64_t)n_elems;
  }
  const int64_t q = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 4;
  const int p = threadIdx.x & 15;
  if (q >= n_quads || p > 12) return;
  Dual X[4][3];
  double ue[24], ve[BI ? 24 : 1];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int n = __ldg(conn + 4 * q + k);
    X[k][0] = Dual(__ldg(gx + n));
    X[k][1] = Dual(__ldg(gy + n));
    X[k][2] = Dual(__ldg(gz + n));
#pragma unroll
    for (int c = 0; c < 6; ++c) {
      ue[6 * k + c] = __ldg(u + 6 * (int64_t)n + c);
      if (BI) ve[BI ? 6 * k + c : 0] = __ldg(vb + 6 * (int64_t)n + c);
    }
  }
  Dual t(__ldg(gt + q));
  if (p < 12) {
#pragma unroll
    for (int k = 0; k < 4; ++k)
#pragma unroll
      for (int a = 0; a < 3; ++a)
        if (3 * k + a == p) X[k][a].d = 1.0;
  } else {
    t.d = 1.0;
  }
  const double Eq = __ldg(gE + n_beams + q);
  const Dual en = quad_energy<BI>(X, t, Eq, __ldg(gnu + n_beams + q), drill_alpha, ue,
                                  *reinterpret_cast<const double(*)[24]>(BI ? ve : ue));
  const double g = -scale * en.d;
  if (p < 12) {
    slot_partial[(2 * (int64_t)n_beams + 4 * q + p / 3) * 3 + (p % 3)] = g;
  } else {
    dC_dt[q] = g;
    // K_e is linear in E_e (SIMP scales the whole elastic tensor): dC/dE = -s u^T K u / E
    // (BI: -s v^T K u / E)
    if (dC_dE) dC_dE[n_beams + q] = -scale * en.v / Eq;
  }
}

// u_e^T K_e u_e of a 3D frame element (reading C1): d_l = T u_e, energy = d_l^T k_loc d_l
// (BI: the bilinear v_e^T K_e u_e with d_l of both states).
template <bool BI>
__global__ void __launch_bounds__(128) beam_grad_kernel(
    int n_beams, const double* __restrict__ gx, const double* __restrict__ gy,
    const double* __restrict__ gz, const int32_t* __restrict__ conn,
    const double* __restrict__ gA, const double* __restrict__ gIy,
    const double* __restrict__ gIz, const double* __restrict__ gJ,
    const double* __restrict__ gE, const double* __restrict__ gG, const double* __restrict__ u,
    const double* __restrict__ vb, double scale, double* __restrict__ slot_partial, double* __restrict__ dC_dE,
    int n_elems, BatchStrides bs) {
  {  // design of a batch (blockIdx.y)
    const int bd = blockIdx.y;
    gx += bd * bs.node;
    gy += bd * bs.node;
    gz += bd * bs.node;
    u += bd * bs.dof;
    if (BI) vb += bd * bs.dof;
    slot_partial += bd * bs.slot;
    if (dC_dE) dC_dE += bd * (int64_t)n_elems;
  }
  const int64_t e = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 3;
  const int p = threadIdx.x & 7;
  if (e >= n_beams || p > 5) return;
  const int ni = __ldg(conn + 2 * e), nj = __ldg(conn + 2 * e + 1);
  Dual Xi[3] = {Dual(__ldg(gx + ni)), Dual(__ldg(gy + ni)), Dual(__ldg(gz + ni))};
  Dual Xj[3] = {Dual(__ldg(gx + nj)), Dual(__ldg(gy + nj)), Dual(__ldg(gz + nj))};
  if (p < 3) Xi[p].d = 1.0; else Xj[p - 3].d = 1.0;
  Dual d[3] = {Xj[0] - Xi[0], Xj[1] - Xi[1], Xj[2] - Xi[2]};
  const Dual L = dsqrt(dot3(d, d));
  const Dual iL = 1.0 / L;
  Dual ex[3] = {d[0] * iL, d[1] * iL, d[2] * iL};
  Dual a[3] = {Dual(0.0), Dual(0.0), Dual(1.0)};
  if (fabs(ex[2].v) > 0.99999999999950000) {
    a[0] = Dual(1.0);
    a[2] = Dual(0.0);
  }
  const Dual ax = dot3(a, ex);
  Dual wv[3] = {a[0] - ax * ex[0], a[1] - ax * ex[1], a[2] - ax * ex[2]};
  const Dual iw = 1.0 / dsqrt(dot3(wv, wv));
  Dual ez[3] = {wv[0] * iw, wv[1] * iw, wv[2] * iw};
  Dual ey[3];
  cross3(ez, ex, ey);
  // local displacements d_l[12] = R applied to each 3-vector of u_e (and of v_e)
  Dual dl[12], dm[12];
  auto localise = [&](const double* __restrict__ uu, Dual (&o)[12]) {
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const int node = (b < 2) ? ni : nj;
      const int off = (b & 1) ? 3 : 0;
      const double g0 = __ldg(uu + 6 * (int64_t)node + off), g1 = __ldg(uu + 6 * (int64_t)node + off + 1),
                   g2 = __ldg(uu + 6 * (int64_t)node + off + 2);
      o[3 * b + 0] = ex[0] * g0 + ex[1] * g1 + ex[2] * g2;
      o[3 * b + 1] = ey[0] * g0 + ey[1] * g1 + ey[2] * g2;
      o[3 * b + 2] = ez[0] * g0 + ez[1] * g1 + ez[2] * g2;
    }
  };
  localise(u, dl);
  if (BI) localise(vb, dm);
  const double E = __ldg(gE + e);
  const double EA = E * __ldg(gA + e), GJ = __ldg(gG + e) * __ldg(gJ + e);
  const double EIy = E * __ldg(gIy + e), EIz = E * __ldg(gIz + e);
  const Dual L2 = L * L, L3 = L2 * L;
  // d_l order: (u, v, w)_i, (thx, thy, thz)_i, (u, v, w)_j, (thx, thy, thz)_j
  const Dual ui = dl[0], vi = dl[1], wi = dl[2], txi = dl[3], tyi = dl[4], tzi = dl[5];
  const Dual uj = dl[6], vj = dl[7], wj = dl[8], txj = dl[9], tyj = dl[10], tzj = dl[11];
  const Dual du = uj - ui, dtx = txj - txi, dv = vi - vj, dw = wi - wj;
  Dual en;
  if (!BI) {
    // quadratic forms of the textbook frame matrix (reading C1), written per sub-problem
    en = (EA / L) * (du * du) + (GJ / L) * (dtx * dtx);
    // x-y bending (v, th_z): [12, 6L, -12, 6L; 6L, 4L^2, -6L, 2L^2; ...] EIz / L^3
    en += (EIz / L3) * (12.0 * (dv * dv) + 12.0 * (L * (dv * (tzi + tzj))) +
                        L2 * (4.0 * (tzi * tzi) + 4.0 * (tzi * tzj) + 4.0 * (tzj * tzj)));
    // x-z bending (w, th_y): signs flipped on the w-th_y coupling
    en += (EIy / L3) * (12.0 * (dw * dw) - 12.0 * (L * (dw * (tyi + tyj))) +
                        L2 * (4.0 * (tyi * tyi) + 4.0 * (tyi * tyj) + 4.0 * (tyj * tyj)));
  } else {
    const Dual duB = dm[6] - dm[0], dtxB = dm[9] - dm[3], dvB = dm[1] - dm[7], dwB = dm[2] - dm[8];
    const Dual tyiB = dm[4], tziB = dm[5], tyjB = dm[10], tzjB = dm[11];
    en = (EA / L) * (duB * du) + (GJ / L) * (dtxB * dtx);
    en += (EIz / L3) * (12.0 * (dvB * dv) + 6.0 * (L * (dvB * (tzi + tzj) + dv * (tziB + tzjB))) +
                        L2 * (4.0 * (tziB * tzi) + 2.0 * (tziB * tzj + tzjB * tzi) + 4.0 * (tzjB * tzj)));
    en += (EIy / L3) * (12.0 * (dwB * dw) - 6.0 * (L * (dwB * (tyi + tyj) + dw * (tyiB + tyjB))) +
                        L2 * (4.0 * (tyiB * tyi) + 2.0 * (tyiB * tyj + tyjB * tyi) + 4.0 * (tyjB * tyj)));
  }
  const double g = -scale * en.d;
  const int node_local = (p < 3) ? 0 : 1;
  slot_partial[(2 * e + node_local) * 3 + (p % 3)] = g;
  if (dC_dE && p == 0) dC_dE[e] = -scale * en.v / E;
}

__global__ void __launch_bounds__(256) node_reduce_kernel(int n_nodes, const int64_t* __restrict__ inc_ptr,
                                                          const int32_t* __restrict__ inc_slot,
                                                          const double* __restrict__ slot_partial,
                                                          double* __restrict__ out, BatchStrides bs) {
  slot_partial += blockIdx.y * bs.slot;
  out += blockIdx.y * 3 * bs.node;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t n = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; n < n_nodes; n += stride) {
    double s0 = 0.0, s1 = 0.0, s2 = 0.0;
    for (int64_t k = inc_ptr[n]; k < inc_ptr[n + 1]; ++k) {
      const int64_t sl = inc_slot[k];
      s0 += slot_partial[3 * sl];
      s1 += slot_partial[3 * sl + 1];
      s2 += slot_partial[3 * sl + 2];
    }
    out[n] = s0;
    out[n_nodes + n] = s1;
    out[2 * (int64_t)n_nodes + n] = s2;
  }
}

}  // namespace

void launch_quad_grad(cudaStream_t s, int n_beams, int n_quads, const double* x, const double* y,
                      const double* z, const int32_t* conn, const double* t, const double* E,
                      const double* nu, double drill_alpha, const double* u, double scale,
                      double* slot_partial, double* dC_dt, double* dC_dE, const BatchStrides& bs,
                      const double* v) {
  if (n_quads <= 0) return;
  const int64_t threads = 16 * (int64_t)n_quads;
  const dim3 grid((unsigned)((threads + 127) / 128), bs.B);
  if (v) {
    quad_grad_kernel<true><<<grid, 128, 0, s>>>(n_beams, n_quads, x, y, z, conn, t, E, nu, drill_alpha, u, v,
                                                scale, slot_partial, dC_dt, dC_dE, n_beams + n_quads, bs);
    SSO_POST_LAUNCH("quad_grad_bilinear_kernel");
  } else {
    quad_grad_kernel<false><<<grid, 128, 0, s>>>(n_beams, n_quads, x, y, z, conn, t, E, nu, drill_alpha, u,
                                                 nullptr, scale, slot_partial, dC_dt, dC_dE, n_beams + n_quads, bs);
    SSO_POST_LAUNCH("quad_grad_kernel");
  }
}

void launch_beam_grad(cudaStream_t s, int n_beams, const double* x, const double* y,
                      const double* z, const int32_t* conn, const double* A, const double* Iy,
                      const double* Iz, const double* J, const double* E, const double* G,
                      const double* u, double scale, double* slot_partial, double* dC_dE, int n_elems,
                      const BatchStrides& bs, const double* v) {
  if (n_beams <= 0) return;
  const int64_t threads = 8 * (int64_t)n_beams;
  const dim3 grid((unsigned)((threads + 127) / 128), bs.B);
  if (v) {
    beam_grad_kernel<true><<<grid, 128, 0, s>>>(n_beams, x, y, z, conn, A, Iy, Iz, J, E, G, u, v, scale,
                                                slot_partial, dC_dE, n_elems, bs);
    SSO_POST_LAUNCH("beam_grad_bilinear_kernel");
  } else {
    beam_grad_kernel<false><<<grid, 128, 0, s>>>(n_beams, x, y, z, conn, A, Iy, Iz, J, E, G, u, nullptr, scale,
                                                 slot_partial, dC_dE, n_elems, bs);
    SSO_POST_LAUNCH("beam_grad_kernel");
  }
}

void launch_node_reduce(cudaStream_t s, int n_nodes, const int64_t* inc_ptr, const int32_t* inc_slot,
                        const double* slot_partial, double* dC_dxyz, const BatchStrides& bs) {
  if (n_nodes <= 0) return;
  int64_t need = ((int64_t)n_nodes + 255) / 256;
  const dim3 grid((unsigned)std::max<int64_t>(1, std::min<int64_t>(need, (int64_t)cg_grid() / bs.B)), bs.B);
  node_reduce_kernel<<<grid, 256, 0, s>>>(n_nodes, inc_ptr, inc_slot, slot_partial, dC_dxyz, bs);
  SSO_POST_LAUNCH("node_reduce_kernel");
}

// SIMP density design variable (Eq. 12):
// E_e = rho_e^P E0_e; G_e = rho_e^P G0_e when given, else E_e / (2 (1 + nu_e)).
__global__ void simp_material_kernel(int ne, const double* __restrict__ rho, double penal,
                                     const double* __restrict__ E0, const double* __restrict__ G0,
                                     const double* __restrict__ nu, double* __restrict__ E,
                                     double* __restrict__ G) {
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < ne; e += gridDim.x * blockDim.x) {
    const double f = pow(rho[e], penal);
    E[e] = f * E0[e];
    G[e] = G0 ? f * G0[e] : E[e] / (2.0 * (1.0 + nu[e]));
  }
}

// dC/drho_e = dC/dE_e * P rho_e^(P-1) E0_e (chain rule of Eq. 12), in place, every design
__global__ void simp_chain_kernel(int ne, int B, const double* __restrict__ rho, double penal,
                                  const double* __restrict__ E0, double* __restrict__ dE) {
  const int64_t n = (int64_t)ne * B;
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x) {
    const int e = (int)(k % ne);
    dE[k] *= penal * pow(rho[e], penal - 1.0) * E0[e];
  }
}

void launch_simp_material(cudaStream_t s, int ne, const double* rho, double penal, const double* E0,
                          const double* G0, const double* nu, double* E, double* G) {
  if (ne <= 0) return;
  simp_material_kernel<<<(ne + 255) / 256, 256, 0, s>>>(ne, rho, penal, E0, G0, nu, E, G);
  SSO_POST_LAUNCH("simp_material_kernel");
}

void launch_simp_chain(cudaStream_t s, int ne, int B, const double* rho, double penal, const double* E0,
                       double* dE) {
  if (ne <= 0) return;
  const int64_t n = (int64_t)ne * B;
  simp_chain_kernel<<<(unsigned)std::min<int64_t>((n + 255) / 256, 4096), 256, 0, s>>>(ne, B, rho, penal, E0, dE);
  SSO_POST_LAUNCH("simp_chain_kernel");
}

}  // namespace sso
