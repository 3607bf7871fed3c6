"""Pins for oracle/grad.py (Eq. 5-6).

  * adjoint gradient == global complex step of C (perturb p by i h,
    re-assemble, complex LU), <= 1e-10 relative: no truncation error on either
    side, so a dropped term or wrong sign anywhere shows;
  * central finite differences (the paper's own check);
  * translation invariance: sum_n dC/dX_n = 0 per axis;
  * rotation identity: sum_n X_n x g_n + 2 sum_n (F_n x u_n + M_n x th_n) = 0
    (s = 1, isotropic supports, Iy = Iz beams);
  * flat plate under in-plane loads: sum_e t_e dC/dt_e = -C (K linear in t);
  * compliance identities f^T u = u^T K u, C(cE) = C / c, C(c f) = c^2 C.
"""
import numpy as np
import pytest

import workloads as W
from oracle import assembly as A, grad as Gd


def _max_rel(a, b):
    return np.abs(a - b).max() / np.abs(b).max()


@pytest.mark.parametrize("make,s", [(lambda: W.tiny_shell(2, 0), 1.0),
                                    (lambda: W.tiny_shell(3, 1), 0.5),
                                    (lambda: W.tiny_beam_grid(0), 1.0)])
def test_adjoint_vs_global_complex_step(make, s):
    P = make()
    u, _, _ = Gd.evaluate(P)
    dX, dt = Gd.adjoint_gradient(P, u, s)
    nn = len(P["x"])
    rng = np.random.default_rng(0)
    nodes = rng.choice(nn, size=min(nn, 4), replace=False)
    for n in nodes:
        for axis in range(3):
            ref = Gd.global_complex_step(P, "xyz", (int(n), axis), s)
            assert abs(dX[axis, n] - ref) <= 1e-10 * max(abs(ref), 1e-6 * np.abs(dX).max())
    for q in range(min(len(dt), 3)):
        ref = Gd.global_complex_step(P, "t", q, s)
        assert abs(dt[q] - ref) <= 1e-10 * max(abs(ref), 1e-6 * np.abs(dt).max())


def test_adjoint_vs_central_fd():
    P = W.tiny_shell(2, 5)
    u, _, _ = Gd.evaluate(P)
    dX, dt = Gd.adjoint_gradient(P, u, 1.0)
    for (n, axis) in [(4, 2), (1, 0), (7, 1)]:
        fd = Gd.central_fd(P, "xyz", (n, axis))
        assert abs(dX[axis, n] - fd) <= 1e-6 * max(abs(fd), 1e-3 * np.abs(dX).max())
    fd = Gd.central_fd(P, "t", 2)
    assert abs(dt[2] - fd) <= 1e-6 * abs(fd)


@pytest.mark.parametrize("make", [lambda: W.tiny_shell(3, 2), lambda: W.tiny_beam_grid(1), W.config1])
def test_translation_and_rotation_identities(make):
    P = make()
    u, _, _ = Gd.evaluate(P)
    dX, _ = Gd.adjoint_gradient(P, u, 1.0)
    scale = np.abs(dX).max()
    assert np.abs(dX.sum(axis=1)).max() <= 1e-9 * scale * len(P["x"])
    X = A.coords(P)
    f = P["f"]
    tot = np.zeros(3)
    for n in range(len(X)):
        tot += np.cross(X[n], dX[:, n])
        tot += 2 * np.cross(f[6 * n:6 * n + 3], u[6 * n:6 * n + 3])
        tot += 2 * np.cross(f[6 * n + 3:6 * n + 6], u[6 * n + 3:6 * n + 6])
    ref = np.abs(X).max() * scale * len(X)
    assert np.abs(tot).max() <= 1e-9 * ref


def test_inplane_thickness_homogeneity():
    n = 3
    x, y = W.grid_nodes(n, 2.0)
    rng = np.random.default_rng(9)
    conn = W.grid_quads(n)
    nq = len(conn)
    f = np.zeros(6 * len(x))
    f[0::6] = rng.uniform(-1e3, 1e3, len(x))
    f[1::6] = rng.uniform(-1e3, 1e3, len(x))
    P = W._problem("flat", x, y, np.zeros_like(x), quad_conn=conn,
                   t=rng.uniform(0.05, 0.2, nq), E=np.full(nq, 30e9), nu=np.full(nq, 0.2),
                   sup_node=[0, n], sup_mask=[W.CLAMPED, W.PINNED], f=f)
    u, _, _ = Gd.evaluate(P)
    C = Gd.compliance(f, u)
    _, dt = Gd.adjoint_gradient(P, u, 1.0)
    assert float(np.dot(P["t"], dt)) == pytest.approx(-C, rel=1e-9)


def test_compliance_identities():
    P = W.tiny_shell(3, 6)
    u, Kb, fb = Gd.evaluate(P)
    C = Gd.compliance(P["f"], u)
    assert C == pytest.approx(float(u @ Kb @ u), rel=1e-10)
    P2 = dict(P)
    P2["E"] = P["E"] * 3.0
    u2, _, _ = Gd.evaluate(P2)
    assert Gd.compliance(P["f"], u2) == pytest.approx(C / 3.0, rel=1e-10)
    P3 = dict(P)
    P3["f"] = P["f"] * 2.5
    u3, _, _ = Gd.evaluate(P3)
    assert Gd.compliance(P3["f"], u3) == pytest.approx(C * 6.25, rel=1e-10)


@pytest.mark.parametrize("make", [lambda: W.tiny_shell(2, 3), lambda: W.tiny_beam_grid(2)])
def test_material_gradient(make):
    """dC/dE_e (SIMP design variable, Eq. 12) against the global complex step,
    and the degree-1 homogeneity of K in E: sum_e E_e dC/dE_e = -C."""
    P = make()
    u, _, _ = Gd.evaluate(P)
    C = Gd.compliance(P["f"], u)
    g = Gd.material_gradient(P, u, 1.0)
    for e in (0, len(g) // 2, len(g) - 1):
        ref = Gd.global_complex_step(P, "E", e, 1.0)
        assert abs(g[e] - ref) <= 1e-10 * max(abs(ref), 1e-6 * np.abs(g).max())
    assert float(np.dot(P["E"], g)) == pytest.approx(-C, rel=1e-10)
    # SIMP chain rule vs complex step through rho (E = rho^P E0)
    rho = np.random.default_rng(1).uniform(0.3, 1.0, len(g))
    E0, penal = P["E"].copy(), 3.0
    Q = dict(P, E=rho ** penal * E0)
    uq, _, _ = Gd.evaluate(Q)
    gq = Gd.simp_gradient(Gd.material_gradient(Q, uq), rho, E0, penal)
    e = 1
    rc = rho.astype(np.complex128)
    rc[e] += 1e-30j
    Qc = dict(P, E=rc ** penal * E0)
    ref = float(np.imag(Gd._solve_C(Qc, A.coords(P).astype(np.complex128),
                                    P["t"].astype(np.complex128), 1.0)) / 1e-30)
    assert gq[e] == pytest.approx(ref, rel=1e-9)


@pytest.mark.parametrize("make", [lambda: W.tiny_shell(2, 4), lambda: W.tiny_beam_grid(3)])
def test_general_adjoint(make):
    """Eq. 5-6 for a non-self-adjoint objective g = c^T u (e.g. a displacement, the
    constraint term of PAPER.md Eq. 9): K lambda = c, dg/dp = -lambda^T (dK/dp) u, checked
    against the complex step of the full solve."""
    P = make()
    u, Kb, fb = Gd.evaluate(P)
    fixed = A.fixed_dofs(P)
    c = np.random.default_rng(8).standard_normal(len(u))
    c[fixed] = 0.0
    free = np.nonzero(~fixed)[0]
    lam = np.zeros_like(u)
    lam[free] = np.linalg.solve(Kb[np.ix_(free, free)], c[free])
    dX, dt, dE = Gd.adjoint_general(P, u, lam)
    nn = len(P["x"])
    for (n, axis) in [(nn // 2, 2), (1, 0), (nn - 2, 1)]:
        ref = Gd.global_complex_step_linear(P, c, "xyz", (n, axis))
        assert abs(dX[axis, n] - ref) <= 1e-9 * max(abs(ref), 1e-6 * np.abs(dX).max())
    if len(dt):
        ref = Gd.global_complex_step_linear(P, c, "t", 1)
        assert abs(dt[1] - ref) <= 1e-9 * max(abs(ref), 1e-6 * np.abs(dt).max())
    ref = Gd.global_complex_step_linear(P, c, "E", 2)
    assert abs(dE[2] - ref) <= 1e-9 * max(abs(ref), 1e-6 * np.abs(dE).max())
    # self-adjoint special case: c = f gives lambda = u and the compliance gradient
    dXc, dtc, _ = Gd.adjoint_general(P, u, u)
    gX, gT = Gd.adjoint_gradient(P, u, 1.0)
    assert np.allclose(dXc, gX, rtol=1e-12, atol=1e-12 * np.abs(gX).max())
