"""Pins for oracle/shell.py (flat MITC-4 shell).

What fixes the element without any implementation to compare against:
  * symmetry, positive semi-definiteness, EXACTLY six rigid-body null modes
    for planar and warped quads (BASELINE.json north_star);
  * each explicit rigid mode (3 translations, 3 rotations) is annihilated;
  * invariance under cyclic relabelling and reversal of the nodes;
  * K(2E) = 2 K(E) bit-exact;
  * membrane and bending patch tests on a distorted patch;
  * Navier series for a simply supported square plate (Kirchhoff and Mindlin),
    thin (t/a = 0.01) and thick (t/a = 0.1, 0.2: pins the transverse shear);
  * complex-step t dK/dt equals the closed form K_m + 3 K_b + K_s + K_d.
"""
import math

import numpy as np
import pytest

import workloads as W
from oracle import assembly as A, grad as Gd, shell

E, NU = 30e9, 0.2


def rand_quad(rng, warp=0.0, scale=1.0):
    base = np.array([[0, 0, 0], [1, 0, 0], [1, 1, 0], [0, 1, 0]], float) * scale
    X = base + rng.uniform(-0.2, 0.2, size=(4, 3)) * scale * np.array([1, 1, 0])
    X[:, 2] += np.array([1, -1, 1, -1]) * warp * scale
    # random rigid placement in 3D
    Q, _ = np.linalg.qr(rng.normal(size=(3, 3)))
    if np.linalg.det(Q) < 0:
        Q[:, 0] *= -1
    return X @ Q.T + rng.normal(size=3)


def rigid_modes(X):
    c = X.mean(axis=0)
    out = []
    for k in range(3):
        r = np.zeros(24)
        r[k::6] = 1.0
        out.append(r)
    for k in range(3):
        w = np.zeros(3)
        w[k] = 1.0
        r = np.zeros(24)
        for i in range(4):
            r[6 * i:6 * i + 3] = np.cross(w, X[i] - c)
            r[6 * i + 3:6 * i + 6] = w
        out.append(r)
    return out


@pytest.mark.parametrize("warp", [0.0, 0.02, 0.1])
@pytest.mark.parametrize("seed", range(4))
def test_null_space_exactly_six(warp, seed):
    rng = np.random.default_rng(seed)
    for scale in (1.0, 0.01):   # h = 1 cm is the C4 element size
        X = rand_quad(rng, warp, scale)
        t = 0.05 + 0.15 * rng.random()
        K = shell.shell_K(X, t, E, NU)
        nrm = np.linalg.norm(K)
        assert np.abs(K - K.T).max() <= 1e-14 * np.abs(K).max()
        d = np.sqrt(np.diag(K))
        S = K / np.outer(d, d)
        ev = np.linalg.eigvalsh(S)
        assert np.all(np.abs(ev[:6]) < 1e-12), ev[:8]
        assert ev[6] > 1e-9, ev[:8]
        for r in rigid_modes(X):
            assert np.linalg.norm(K @ r) <= 1e-12 * nrm * np.linalg.norm(r)


def test_relabel_invariance_and_E_scaling():
    rng = np.random.default_rng(11)
    X = rand_quad(rng, 0.05)
    K = shell.shell_K(X, 0.1, E, NU)
    for perm in ([1, 2, 3, 0], [2, 3, 0, 1], [3, 2, 1, 0], [0, 3, 2, 1]):
        Kp = shell.shell_K(X[perm], 0.1, E, NU)
        idx = np.array([6 * p + c for p in perm for c in range(6)])
        assert np.abs(Kp - K[np.ix_(idx, idx)]).max() <= 1e-12 * np.abs(K).max()
    assert np.array_equal(shell.shell_K(X, 0.1, 2 * E, NU), 2 * shell.shell_K(X, 0.1, E, NU))


def test_thickness_derivative_closed_form():
    rng = np.random.default_rng(3)
    X = rand_quad(rng, 0.05)
    t = 0.12
    Kc = shell.shell_K(X, t + 1j * 1e-30, E, NU)
    dK = np.imag(Kc) / 1e-30
    ref = shell.shell_t_dKdt(X, t, E, NU) / t
    assert np.abs(dK - ref).max() <= 1e-12 * np.abs(ref).max()


def _patch():
    # 4-quad distorted patch on [0, 2]^2, interior node 4 moved off-centre
    pts = np.array([[0, 0], [1, 0], [2, 0], [0, 1], [1.13, 0.91], [2, 1], [0, 2], [1, 2], [2, 2]],
                   float)
    conn = np.array([[0, 1, 4, 3], [1, 2, 5, 4], [3, 4, 7, 6], [4, 5, 8, 7]], np.int32)
    return pts, conn


def _patch_solve(prescribed):
    """Solve the patch with all 8 boundary nodes fully prescribed (values from
    `prescribed(x, y)` -> 6-vector) and return interior-node DOFs and exact."""
    pts, conn = _patch()
    nn = len(pts)
    P = W._problem("patch", pts[:, 0], pts[:, 1], np.zeros(nn), quad_conn=conn,
                   t=np.full(4, 0.1), E=np.full(4, E), nu=np.full(4, NU),
                   sup_node=[0], sup_mask=[W.CLAMPED], f=np.zeros(6 * nn))
    dok = A.assemble_dok(P)
    K = A.dense_from_dok(dok, 6 * nn)
    b = [k for k in range(nn) if k != 4]
    bd = [6 * k + c for k in b for c in range(6)]
    idof = [24 + c for c in range(6)]
    ub = np.concatenate([prescribed(*pts[k]) for k in b])
    ui = np.linalg.solve(K[np.ix_(idof, idof)], -K[np.ix_(idof, bd)] @ ub)
    return ui, prescribed(*pts[4])


def test_membrane_patch():
    a0, a1, a2, b0, b1, b2 = 1e-3, 2e-3, -1.5e-3, 0.5e-3, 0.7e-3, 1.1e-3

    def field(x, y):
        u = a0 + a1 * x + a2 * y
        v = b0 + b1 * x + b2 * y
        om = 0.5 * (b1 - a2)           # theta_z = omega = 1/2 (v,x - u,y)
        return np.array([u, v, 0.0, 0.0, 0.0, om])

    ui, ex = _patch_solve(field)
    assert np.abs(ui - ex).max() <= 1e-10 * np.abs(ex).max()


def test_bending_patch():
    a, b, c = 1e-3, -2e-3, 0.7e-3

    def field(x, y):
        w = 0.5 * (a * x * x + b * y * y + c * x * y)
        wx = a * x + 0.5 * c * y
        wy = b * y + 0.5 * c * x
        return np.array([0.0, 0.0, w, wy, -wx, 0.0])   # th_x = w,y ; th_y = -w,x

    ui, ex = _patch_solve(field)
    assert np.abs(ui - ex).max() <= 1e-10 * np.abs(ex).max()


def _navier_series(q, a, D, ks_G_t=None, terms=101):
    s = 0.0
    for m in range(1, 2 * terms, 2):
        for n in range(1, 2 * terms, 2):
            wmn = 16 * q / (math.pi ** 6 * D * m * n * (m * m + n * n) ** 2)
            if ks_G_t is not None:
                k2 = (m * math.pi / a) ** 2 + (n * math.pi / a) ** 2
                wmn *= 1 + D * k2 / ks_G_t
            s += wmn * (-1) ** ((m - 1) // 2 + (n - 1) // 2)
    return s * a ** 4


def _navier_center(n, a, t, Ep, nu, q):
    """Centre deflection of the oracle's hard simply supported square plate
    (w = 0 on every edge, tangential rotation fixed, u = v = 0)."""
    x, y = W.grid_nodes(n, a)
    conn = W.grid_quads(n)
    nq = len(conn)
    f = W.lumped_vertical_load(x, y, np.zeros_like(x), conn, q)
    sn, sm = [], []
    for k in range(len(x)):
        m = 0
        if x[k] in (0.0, a):
            m |= 0b001111        # u, v, w, th_x
        if y[k] in (0.0, a):
            m |= 0b010111        # u, v, w, th_y
        if m:
            sn.append(k)
            sm.append(m)
    P = W._problem("navier", x, y, np.zeros_like(x), quad_conn=conn, t=np.full(nq, t),
                   E=np.full(nq, Ep), nu=np.full(nq, nu), sup_node=sn, sup_mask=sm, f=f)
    u, _, _ = Gd.evaluate(P)
    return -u[6 * ((n // 2) * (n + 1) + n // 2) + 2]


@pytest.mark.slow
def test_navier_plate():
    n, a, t, Ep, nu, q = 32, 1.0, 0.01, 1e9, 0.3, 1.0
    wc = _navier_center(n, a, t, Ep, nu, q)
    D = Ep * t ** 3 / (12 * (1 - nu ** 2))
    wk = _navier_series(q, a, D)
    assert wk / (q * a ** 4 / D) == pytest.approx(0.0040624, rel=1e-4)
    wm = _navier_series(q, a, D, ks_G_t=5 / 6 * Ep / (2 * (1 + nu)) * t)
    assert abs(wc / wk - 1) < 0.01
    assert abs(wc / wm - 1) < 0.005


@pytest.mark.slow
@pytest.mark.parametrize("t", [0.1, 0.2])
def test_navier_thick_plate_shear(t):
    """Thick-plate pin of the MITC-4 transverse shear (§2.2.1, SURVEY
    §8(c) C2(f), C10): at t/a = 0.1 and 0.2 the Mindlin shear term is 2-8 % of the
    centre deflection (at t/a = 0.01 it is 5e-4), so k_s, G = E/(2(1+nu)) and the
    J^-1 mapping of the tied covariant strains are all visible.  The hard simply
    supported Mindlin plate has the closed-form Navier series with modal factor
    (1 + D k^2 / (k_s G t)), k^2 = (m pi/a)^2 + (n pi/a)^2; the 32x32 oracle mesh must
    be within 0.3 % of it, while the same series with k_s = 1 (a plausible wrong
    shear factor) must be further than 0.5 % away (the pin discriminates)."""
    n, a, Ep, nu, q = 32, 1.0, 1e9, 0.3, 1.0
    wc = _navier_center(n, a, t, Ep, nu, q)
    D = Ep * t ** 3 / (12 * (1 - nu ** 2))
    G = Ep / (2 * (1 + nu))
    wm = _navier_series(q, a, D, ks_G_t=5 / 6 * G * t)
    wk = _navier_series(q, a, D)
    w_ks1 = _navier_series(q, a, D, ks_G_t=1.0 * G * t)
    assert wm / wk - 1 > 0.02                   # the shear term is large here
    assert abs(wc / wm - 1) < 0.003, wc / wm
    assert abs(wm / w_ks1 - 1) > 0.005          # k_s = 1 would fail the 0.3 % bar


@pytest.mark.parametrize("seed", range(6))
def test_constant_transverse_shear_energy(seed):
    """Closed-form energy of a constant transverse-shear state on a distorted flat
    quad: with w = c1 x + c2 y and constant rotations
    (th_x, th_y) = (a, b) there is no membrane strain, no curvature and no drilling
    strain, and MITC-4's tied covariant strains reproduce the constant Cartesian
    shear (gamma_xz, gamma_yz) = (c1 + b, c2 - a) exactly on any bilinear quad
    (gamma_xi = gamma . x_xi is linear in eta along xi-lines, and J^-1 J = I).
    So 1/2 u^T K u = 1/2 k_s G t A (gamma_xz^2 + gamma_yz^2) to rounding.  This
    fixes k_s, G, the shear sign convention beta = (th_y, -th_x) and the J^-1
    mapping on non-rectangular elements (a transposed J^-1 fails it)."""
    rng = np.random.default_rng(100 + seed)
    base = np.array([[0, 0], [1, 0], [1, 1], [0, 1]], float)
    P2 = base + rng.uniform(-0.25, 0.25, size=(4, 2))
    th = rng.uniform(0, 2 * math.pi)
    Rz = np.array([[math.cos(th), -math.sin(th)], [math.sin(th), math.cos(th)]])
    P2 = P2 @ Rz.T * rng.uniform(0.01, 3.0) + rng.normal(size=2)
    X = np.column_stack([P2, np.zeros(4)])
    t = rng.uniform(0.05, 0.3)
    c1, c2, a, b = rng.normal(size=4)
    u = np.zeros(24)
    for i in range(4):
        u[6 * i + 2] = c1 * X[i, 0] + c2 * X[i, 1]
        u[6 * i + 3] = a
        u[6 * i + 4] = b
    K = shell.shell_K(X, t, E, NU)
    x, y = X[:, 0], X[:, 1]
    area = 0.5 * abs((x[2] - x[0]) * (y[3] - y[1]) - (x[3] - x[1]) * (y[2] - y[0]))
    G = E / (2 * (1 + NU))
    ref = 0.5 * (5 / 6) * G * t * area * ((c1 + b) ** 2 + (c2 - a) ** 2)
    assert 0.5 * u @ K @ u == pytest.approx(ref, rel=1e-11)
