"""Oracle: design-dependent area loads and their share of the adjoint gradient
(test infrastructure only).

PAPER.md:216-220 (Eq. 6) keeps the load term: dg/dp = dg/dp|explicit -
lambda^T (dK/dp u - df/dp).  This build's default holds f fixed (reading c3);
with a design-dependent load f(p) and the compliance g = s f^T u (lambda = s u)
the gradient becomes

    dC/dp = s (2 u^T df/dp - u^T dK/dp u)                              (reading c17)

The load model (reading c17, the area load of reading c11 made part of the
method): every quad e carries a load per unit area (q_e + w_e t_e) in the fixed
direction d (w_e = unit weight, i.e. rho g, so w_e t_e is self-weight), lumped
to its 4 nodes equally with the area A_e = 1/2 |(X3 - X1) x (X4 - X2)|:

    f_n[0:3] += d (q_e + w_e t_e) A_e / 4     for each node n of quad e.

df/dp is taken by complex step on the element load routine (exact to roundoff).
Pins (tests/test_oracle_loads.py): the total load of a flat rectangle equals
(q + w t) x area in closed form; the load matches the independent lumping of
workloads.lumped_vertical_load; the gradient equals the global complex step of
the full solve with f recomputed at every perturbed design.
"""
from __future__ import annotations

import numpy as np

from . import assembly as A
from . import grad as Gd
from . import solve as S


def element_area_load(Xe, t_e, q_e, w_e, d):
    """[4, 3] translational nodal forces of one quad (complex-capable)."""
    c = np.cross(Xe[2] - Xe[0], Xe[3] - Xe[1])
    area = 0.5 * np.sqrt(np.sum(c * c))
    return np.outer(np.ones(4), np.asarray(d)) * ((q_e + w_e * t_e) * area / 4.0)


def area_load(P, q, w, d, X=None, t=None):
    """Full load vector [6 n_nodes] of the area loads (quads, ascending order)."""
    if X is None:
        X = A.coords(P)
    if t is None:
        t = P["t"]
    dt = np.complex128 if (np.iscomplexobj(X) or np.iscomplexobj(t)) else np.float64
    f = np.zeros(6 * len(P["x"]), dtype=dt)
    for e, nodes in enumerate(P["quad_conn"]):
        fe = element_area_load(X[list(nodes)], t[e], q[e], w[e], d)
        for k, n in enumerate(nodes):
            f[6 * n:6 * n + 3] += fe[k]
    return f


def load_gradient_term(P, v, q, w, d, X=None):
    """v^T df/dp for the coordinates [3, n_nodes] and thicknesses [n_quads], by
    complex step on element_area_load (the term Eq. 6 adds, with v = lambda)."""
    if X is None:
        X = A.coords(P)
    t = P["t"]
    gX = np.zeros((3, len(P["x"])))
    gt = np.zeros(len(t))
    h = Gd.H_CS
    for e, nodes in enumerate(P["quad_conn"]):
        nodes = list(nodes)
        ve = np.array([v[6 * n:6 * n + 3] for n in nodes])
        Xe = X[nodes].astype(np.complex128)
        for k in range(4):
            for a in range(3):
                Xp = Xe.copy()
                Xp[k, a] += 1j * h
                dfe = np.imag(element_area_load(Xp, t[e], q[e], w[e], d)) / h
                gX[a, nodes[k]] += float(np.sum(ve * dfe))
        dfe = np.imag(element_area_load(Xe, t[e] + 1j * h, q[e], w[e], d)) / h
        gt[e] = float(np.sum(ve * dfe))
    return gX, gt


def compliance_gradient(P, u, q, w, d, s=1.0):
    """dC/dX [3, n], dC/dt [n_quads] with the design-dependent load:
    s (2 u^T df/dp - u^T dK/dp u)."""
    dX, dt = Gd.adjoint_gradient(P, u, s)
    lX, lt = load_gradient_term(P, u, q, w, d)
    return dX + 2.0 * s * lX, dt + 2.0 * s * lt


def evaluate(P, q, w, d):
    """u for f = P['f'] + area_load (dense Cholesky); returns (u, f_total)."""
    f = P["f"] + area_load(P, q, w, d)
    u, _, _ = Gd.evaluate(dict(P, f=f))
    return u, f


def global_complex_step(P, q, w, d, kind, index, s=1.0):
    """dC/dp of C = s f(p)^T u(p) with the load recomputed at the perturbed design."""
    X = A.coords(P).astype(np.complex128)
    t = P["t"].astype(np.complex128)
    h = Gd.H_CS
    if kind == "xyz":
        X[index[0], index[1]] += 1j * h
    else:
        t[index] += 1j * h
    nd = 6 * len(P["x"])
    f = P["f"].astype(np.complex128) + area_load(P, q, w, d, X, t)
    K = A.dense_from_dok(A.assemble_dok(P, X, t), nd, dtype=np.complex128)
    fixed = A.fixed_dofs(P)
    Kbc, fbc = A.apply_supports_dense(K, f, fixed)
    free = np.nonzero(~fixed)[0]
    u = np.zeros(nd, dtype=np.complex128)
    u[free] = S.solve_dense_lu(Kbc[np.ix_(free, free)], fbc[free])
    return float(np.imag(s * np.dot(fbc, u)) / h)
