"""Oracle: flat 4-node MITC-4 shell element, 24x24 (test infrastructure only).

PAPER.md:44 and :75-82 name the element ("quad shell elements based on
MITC-4", `element_K_quad_local`, attributes a_quad = (x, y, z, t, E, nu,
kappa_x, kappa_y)) but fix none of its details.  This file follows SURVEY.md
§8(c) C2 (a)-(h) step by step — DESIGN.md reading c4 — in that order:

  (a) intrinsic frame from the diagonals, local planar coords, warp offsets h_i
  (b) bilinear geometry, 2x2 Gauss points in the order (-,-), (+,-), (+,+), (-,+)
  (c) rigid-offset warping correction W_i (u_P = u - h th_y, v_P = v + h th_x)
  (d) plane-stress membrane
  (e) Mindlin bending (beta_x = th_y, beta_y = -th_x)
  (f) MITC-4 (Dvorkin-Bathe) assumed transverse shear, tying points A, B, C, D
  (g) coupled drilling penalty gamma_d = alpha_d G, alpha_d = 1e-3
  (h) K_e = T^T W^T K_loc W T; kappa_x = kappa_y = 1 (reading c5)

Complex-step safe: norms are sqrt(sum(v*v)), branches only on real parts.

Pins: tests/test_oracle_shell.py — symmetry, PSD, exactly six null modes
(planar and warped), explicit rigid modes, relabel invariance, K(2E) = 2K(E),
membrane and bending patch tests, Navier plate series (Kirchhoff and Mindlin),
t dK/dt = K_m + 3K_b + K_s + K_d, and the paper's barrel-arch values
(PAPER.md:145, 252).
"""
from __future__ import annotations

import math
import numpy as np

GAUSS = 1.0 / math.sqrt(3.0)
# (xi, eta) of the 2x2 Gauss points, order (-,-), (+,-), (+,+), (-,+); weight 1
GAUSS_PTS = [(-GAUSS, -GAUSS), (GAUSS, -GAUSS), (GAUSS, GAUSS), (-GAUSS, GAUSS)]
# natural coordinates of the 4 nodes
XI_N = [-1.0, 1.0, 1.0, -1.0]
ETA_N = [-1.0, -1.0, 1.0, 1.0]
K_SHEAR = 5.0 / 6.0
ALPHA_DRILL = 1e-3

# local DOF offsets within a node block
U, V, W_, TX, TY, TZ = 0, 1, 2, 3, 4, 5


def _dot(a, b):
    return a[0] * b[0] + a[1] * b[1] + a[2] * b[2]


def _cross(a, b):
    return np.array([a[1] * b[2] - a[2] * b[1],
                     a[2] * b[0] - a[0] * b[2],
                     a[0] * b[1] - a[1] * b[0]], dtype=np.result_type(a, b))


def shell_frame(X):
    """C2(a): centroid c, normal n = (X3-X1) x (X4-X2), e3 = n/|n|;
    d = (X2-X1) - ((X2-X1).e3) e3, e1 = d/|d|, e2 = e3 x e1; R = [e1; e2; e3].
    Returns R, local (x_i, y_i), warp offsets h_i.  Raises on |n| = 0."""
    X = np.asarray(X)
    c = (X[0] + X[1] + X[2] + X[3]) / 4.0
    n = _cross(X[2] - X[0], X[3] - X[1])
    nn = np.sqrt(_dot(n, n))
    if np.real(nn) <= 0.0:
        raise ValueError("degenerate quad: zero normal")
    e3 = n / nn
    d = (X[1] - X[0]) - _dot(X[1] - X[0], e3) * e3
    e1 = d / np.sqrt(_dot(d, d))
    e2 = _cross(e3, e1)
    R = np.array([e1, e2, e3])
    xl = [_dot(X[i] - c, e1) for i in range(4)]
    yl = [_dot(X[i] - c, e2) for i in range(4)]
    h = [_dot(X[i] - c, e3) for i in range(4)]
    return R, xl, yl, h


def shape_derivs(xl, yl, xi, eta):
    """C2(b): N_i = 1/4 (1 + xi_i xi)(1 + eta_i eta); J = [[x_xi, y_xi], [x_eta, y_eta]];
    [N_i,x; N_i,y] = J^-1 [N_i,xi; N_i,eta].  Returns (N, dNdx, dNdy, detJ, Jinv)."""
    N = [0.25 * (1 + XI_N[i] * xi) * (1 + ETA_N[i] * eta) for i in range(4)]
    dxi = [0.25 * XI_N[i] * (1 + ETA_N[i] * eta) for i in range(4)]
    deta = [0.25 * ETA_N[i] * (1 + XI_N[i] * xi) for i in range(4)]
    x_xi = sum(dxi[i] * xl[i] for i in range(4))
    y_xi = sum(dxi[i] * yl[i] for i in range(4))
    x_eta = sum(deta[i] * xl[i] for i in range(4))
    y_eta = sum(deta[i] * yl[i] for i in range(4))
    detJ = x_xi * y_eta - y_xi * x_eta
    # J^-1 = 1/det [[y_eta, -y_xi], [-x_eta, x_xi]]
    Jinv = [[y_eta / detJ, -y_xi / detJ], [-x_eta / detJ, x_xi / detJ]]
    dNdx = [Jinv[0][0] * dxi[i] + Jinv[0][1] * deta[i] for i in range(4)]
    dNdy = [Jinv[1][0] * dxi[i] + Jinv[1][1] * deta[i] for i in range(4)]
    return N, dNdx, dNdy, detJ, Jinv


def _plane_D(scale, nu):
    return scale * np.array([[1.0, nu, 0.0], [nu, 1.0, 0.0], [0.0, 0.0, (1.0 - nu) / 2.0]])


def shell_local_parts(X, t, E, nu, alpha_d=ALPHA_DRILL):
    """C2(a)-(g): the four local 24x24 parts (K_m, K_b, K_s, K_d), on projected
    local DOFs (u, v, w, th_x, th_y, th_z) per node, plus R, h and area A_e."""
    R, xl, yl, h = shell_frame(X)
    dt = np.result_type(np.asarray(X), t, E, nu, np.float64)
    Km = np.zeros((24, 24), dtype=dt)
    Kb = np.zeros((24, 24), dtype=dt)
    Ks = np.zeros((24, 24), dtype=dt)
    Kd = np.zeros((24, 24), dtype=dt)
    G = E / (2.0 * (1.0 + nu))
    Dm = _plane_D(E * t / (1.0 - nu * nu), nu)
    Db = _plane_D(E * t ** 3 / (12.0 * (1.0 - nu * nu)), nu)
    ds = K_SHEAR * G * t

    # C2(f) tying-point covariant shear strains as rows over the 24 DOFs.
    # beta_i = (th_y_i, -th_x_i); x_i = (x_i, y_i).
    def row_gamma(n_plus, n_minus):
        """1/2 (w_plus - w_minus) + 1/2 (beta_plus + beta_minus) . 1/2 (x_plus - x_minus)"""
        row = np.zeros(24, dtype=dt)
        dx = 0.5 * (xl[n_plus] - xl[n_minus])
        dy = 0.5 * (yl[n_plus] - yl[n_minus])
        row[6 * n_plus + W_] += 0.5
        row[6 * n_minus + W_] += -0.5
        for nd in (n_plus, n_minus):
            # 1/2 beta_nd . (dx, dy) with beta = (th_y, -th_x)
            row[6 * nd + TY] += 0.5 * dx
            row[6 * nd + TX] += -0.5 * dy
        return row

    g_xi_A = row_gamma(2, 3)   # A = (0, 1):  1/2(w3 - w4) + 1/2(b3 + b4).1/2(x3 - x4)
    g_xi_C = row_gamma(1, 0)   # C = (0,-1):  1/2(w2 - w1) + 1/2(b1 + b2).1/2(x2 - x1)
    g_eta_D = row_gamma(2, 1)  # D = (1, 0):  1/2(w3 - w2) + 1/2(b2 + b3).1/2(x3 - x2)
    g_eta_B = row_gamma(3, 0)  # B = (-1,0):  1/2(w4 - w1) + 1/2(b1 + b4).1/2(x4 - x1)

    area = 0.0
    for (xi, eta) in GAUSS_PTS:
        N, dNdx, dNdy, detJ, Jinv = shape_derivs(xl, yl, xi, eta)
        if np.real(detJ) <= 0.0:
            raise ValueError("degenerate quad: det J <= 0 at a Gauss point")
        area = area + detJ
        # (d) membrane B (3 x 24)
        Bm = np.zeros((3, 24), dtype=dt)
        for i in range(4):
            Bm[0, 6 * i + U] = dNdx[i]
            Bm[1, 6 * i + V] = dNdy[i]
            Bm[2, 6 * i + U] = dNdy[i]
            Bm[2, 6 * i + V] = dNdx[i]
        Km += Bm.T @ Dm @ Bm * detJ
        # (e) bending B (3 x 24) on (th_x, th_y)
        Bb = np.zeros((3, 24), dtype=dt)
        for i in range(4):
            Bb[0, 6 * i + TY] = dNdx[i]
            Bb[1, 6 * i + TX] = -dNdy[i]
            Bb[2, 6 * i + TX] = -dNdx[i]
            Bb[2, 6 * i + TY] = dNdy[i]
        Kb += Bb.T @ Db @ Bb * detJ
        # (f) assumed covariant shear, then Cartesian via J^-1
        g_xi = 0.5 * (1 + eta) * g_xi_A + 0.5 * (1 - eta) * g_xi_C
        g_eta = 0.5 * (1 + xi) * g_eta_D + 0.5 * (1 - xi) * g_eta_B
        Bs = np.zeros((2, 24), dtype=dt)
        Bs[0] = Jinv[0][0] * g_xi + Jinv[0][1] * g_eta
        Bs[1] = Jinv[1][0] * g_xi + Jinv[1][1] * g_eta
        Ks += ds * (Bs.T @ Bs) * detJ

    # (g) drilling: omega_c = 1/2 (v,x - u,y) at the centre; b_i = e_thz_i - b_omega
    _, dNdx0, dNdy0, _, _ = shape_derivs(xl, yl, 0.0, 0.0)
    b_omega = np.zeros(24, dtype=dt)
    for i in range(4):
        b_omega[6 * i + U] = -0.5 * dNdy0[i]
        b_omega[6 * i + V] = 0.5 * dNdx0[i]
    gamma_d = alpha_d * G
    for i in range(4):
        b = -b_omega.copy()
        b[6 * i + TZ] += 1.0
        Kd += gamma_d * t * (area / 4.0) * np.outer(b, b)
    return Km, Kb, Ks, Kd, R, h, area


def shell_transform(R, h):
    """C2(c)+(h): the 24x24 map Q = W T from global DOFs to projected local DOFs.
    T = blockdiag over 8 of R; W_i = I_6 with W[u, th_y] = -h_i, W[v, th_x] = +h_i."""
    dt = np.result_type(R, np.asarray(h))
    T = np.zeros((24, 24), dtype=dt)
    for b in range(8):
        T[3 * b:3 * b + 3, 3 * b:3 * b + 3] = R
    Wm = np.eye(24, dtype=dt)
    for i in range(4):
        Wm[6 * i + U, 6 * i + TY] = -h[i]
        Wm[6 * i + V, 6 * i + TX] = h[i]
    return Wm @ T


def shell_K(X, t, E, nu, alpha_d=ALPHA_DRILL):
    """Global 24x24 element stiffness K_e = T^T W^T (K_m + K_b + K_s + K_d) W T
    (SURVEY.md §8(c) C2(h)); node-major, component-minor global DOFs."""
    Km, Kb, Ks, Kd, R, h, _ = shell_local_parts(X, t, E, nu, alpha_d)
    Q = shell_transform(R, h)
    return Q.T @ (Km + Kb + Ks + Kd) @ Q


def shell_t_dKdt(X, t, E, nu, alpha_d=ALPHA_DRILL):
    """t dK_e/dt = T^T W^T (K_m + 3 K_b + K_s + K_d) W T (C2(h), exact)."""
    Km, Kb, Ks, Kd, R, h, _ = shell_local_parts(X, t, E, nu, alpha_d)
    Q = shell_transform(R, h)
    return Q.T @ (Km + 3.0 * Kb + Ks + Kd) @ Q
