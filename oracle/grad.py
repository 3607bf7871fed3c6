"""Oracle: compliance and its adjoint gradient (test infrastructure only).

PAPER.md:212-221 (Eqs. 5-6): K^T lambda = dg/du^T;
dg/dp = dg/dp|explicit - lambda^T (dK/dp u - df/dp).  For compliance
g = s f^T u with f fixed (df/dp = 0, reading c3) and K symmetric, the adjoint
is lambda = s u (no second solve) and Eq. 6 reduces to

    dC/dp = - s * sum_e u_e^T (dK_e/dp) u_e

with s = 1 for compliance f^T u and s = 1/2 for the paper's strain energy
0.5 f^T u (reading c2).  u_e is taken from the full u
(zeros at supports).  dK_e/dp is computed by complex step on the same loop
code as K_e: dK_e/dp = Im K_e(p + i h) / h, h = 1e-30 (exact to roundoff).

Also here, for the pins: the global complex-step derivative of C (perturb p by
i h, re-assemble, complex dense LU solve) and central finite differences
(the paper's own validation method).
"""
from __future__ import annotations

import numpy as np

from . import assembly as A
from . import solve as S

H_CS = 1e-30


def compliance(f, u, s=1.0):
    """C = s f^T u."""
    return s * float(np.dot(f, u))


def evaluate(P, solver="cholesky", rtol=1e-12, X=None, t=None):
    """Forward FEA: DOK assembly -> supports -> solve.  Returns (u, K_bc, f_bc)."""
    nd = 6 * len(P["x"])
    dok = A.assemble_dok(P, X, t)
    fixed = A.fixed_dofs(P)
    if solver == "cholesky":
        K = A.dense_from_dok(dok, nd)
        Kbc, fbc = A.apply_supports_dense(K, P["f"], fixed)
        u = S.solve_dense_cholesky(Kbc, fbc, fixed)
        return u, Kbc, fbc
    if solver == "pcg":
        import scipy.sparse as sp
        row_ptr, col_idx, vals = A.csr_from_dok(dok, nd)
        vals = A.apply_supports_csr(row_ptr, col_idx, vals, fixed)
        Kc = sp.csr_matrix((vals, col_idx, row_ptr), shape=(nd, nd))
        fbc = P["f"].copy()
        fbc[fixed] = 0.0
        diag = Kc.diagonal()
        u, info = S.pcg(Kc, fbc, 1.0 / diag, rtol=rtol)
        return u, Kc, fbc
    raise ValueError(solver)


def element_dK_dcoord(P, e, node_local, axis, X=None):
    """dK_e / dX_{node, axis} by complex step on the element routine."""
    if X is None:
        X = A.coords(P)
    Xc = X.astype(np.complex128)
    n = A.element_nodes(P, e)[node_local]
    Xc[n, axis] += 1j * H_CS
    return np.imag(A.element_K(P, e, Xc)) / H_CS


def element_dK_dt(P, e, X=None):
    """dK_e / dt_e by complex step (quads only)."""
    nb = A.n_beams(P)
    tc = P["t"].astype(np.complex128)
    tc[e - nb] += 1j * H_CS
    return np.imag(A.element_K(P, e, X, tc)) / H_CS


def adjoint_gradient(P, u, s=1.0):
    """dC/dX [3, n_nodes] and dC/dt [n_quads] by the reduced Eq. 6 above; node sums
    run over elements in ascending order."""
    nn = len(P["x"])
    nb, nq = A.n_beams(P), A.n_quads(P)
    X = A.coords(P)
    dX = np.zeros((3, nn))
    dt = np.zeros(nq)
    for e in range(nb + nq):
        nodes = A.element_nodes(P, e)
        ue = u[A.element_dofs(nodes)]
        for il, n in enumerate(nodes):
            for axis in range(3):
                dK = element_dK_dcoord(P, e, il, axis, X)
                dX[axis, n] += -s * float(ue @ dK @ ue)
        if e >= nb:
            dK = element_dK_dt(P, e, X)
            dt[e - nb] = -s * float(ue @ dK @ ue)
    return dX, dt


def element_grad(P, e, u, s=1.0, X=None):
    """Per-element contributions: ([k, 3] coordinate partials, dC/dt_e or None)."""
    if X is None:
        X = A.coords(P)
    nb = A.n_beams(P)
    nodes = A.element_nodes(P, e)
    ue = u[A.element_dofs(nodes)]
    out = np.zeros((len(nodes), 3))
    for il in range(len(nodes)):
        for axis in range(3):
            dK = element_dK_dcoord(P, e, il, axis, X)
            out[il, axis] = -s * float(ue @ dK @ ue)
    g_t = None
    if e >= nb:
        dK = element_dK_dt(P, e, X)
        g_t = -s * float(ue @ dK @ ue)
    return out, g_t


def element_dK_dE(P, e, X=None):
    """dK_e / dE_e by complex step (any element).  The whole elastic tensor of the
    element scales with E_e (SIMP, Eq. 12): an explicitly given G scales by
    the same factor."""
    Pc = dict(P)
    Pc["E"] = P["E"].astype(np.complex128)
    Pc["E"][e] += 1j * H_CS
    if P.get("G") is not None:
        Pc["G"] = P["G"].astype(np.complex128)
        Pc["G"][e] *= Pc["E"][e] / P["E"][e]
    return np.imag(A.element_K(Pc, e, X)) / H_CS


def material_gradient(P, u, s=1.0):
    """dC/dE_e = -s u_e^T (dK_e/dE_e) u_e for every element (beams first, then quads):
    the adjoint gradient of PAPER.md Eq. 6 with respect to the element modulus, the
    design variable of SIMP (Eq. 12: E_j = p_T,j^P E_*,j)."""
    nb, nq = A.n_beams(P), A.n_quads(P)
    X = A.coords(P)
    out = np.zeros(nb + nq)
    for e in range(nb + nq):
        ue = u[A.element_dofs(A.element_nodes(P, e))]
        out[e] = -s * float(ue @ element_dK_dE(P, e, X) @ ue)
    return out


def simp_gradient(dC_dE, rho, E0, penal):
    """SIMP chain rule (Eq. 12): E = rho^P E0 -> dC/drho = dC/dE * P rho^(P-1) E0."""
    return dC_dE * penal * rho ** (penal - 1.0) * E0


def _solve_C(P, X, t, s):
    nd = 6 * len(P["x"])
    dok = A.assemble_dok(P, X, t)
    dtp = np.complex128 if (np.iscomplexobj(X) or np.iscomplexobj(t)) else np.float64
    K = A.dense_from_dok(dok, nd, dtype=dtp)
    fixed = A.fixed_dofs(P)
    Kbc, fbc = A.apply_supports_dense(K, P["f"].astype(dtp), fixed)
    free = np.nonzero(~fixed)[0]
    u = np.zeros(nd, dtype=dtp)
    u[free] = S.solve_dense_lu(Kbc[np.ix_(free, free)], fbc[free])
    return s * np.dot(P["f"], u)


def global_complex_step(P, kind, index, s=1.0):
    """dC/dp for p = coordinate (kind='xyz', index=(node, axis)), thickness
    (kind='t', index=quad) or modulus (kind='E', index=element) by perturbing p with
    i h, re-assembling and solving the complex system with dense LU (loads held
    fixed, reading c3)."""
    X = A.coords(P).astype(np.complex128)
    t = P["t"].astype(np.complex128)
    if kind == "xyz":
        X[index[0], index[1]] += 1j * H_CS
    elif kind == "t":
        t[index] += 1j * H_CS
    else:
        Pc = dict(P)
        Pc["E"] = P["E"].astype(np.complex128)
        Pc["E"][index] += 1j * H_CS
        return float(np.imag(_solve_C(Pc, X, t, s)) / H_CS)
    return float(np.imag(_solve_C(P, X, t, s)) / H_CS)


def central_fd(P, kind, index, s=1.0, rel_step=1e-6):
    """Central finite difference with step 1e-6 (1 + |p|)."""
    X = A.coords(P).copy()
    t = P["t"].copy()
    if kind == "xyz":
        p0 = X[index[0], index[1]]
    else:
        p0 = t[index]
    hstep = rel_step * (1.0 + abs(p0))
    vals = []
    for sgn in (1.0, -1.0):
        Xp, tp = X.copy(), t.copy()
        if kind == "xyz":
            Xp[index[0], index[1]] = p0 + sgn * hstep
        else:
            tp[index] = p0 + sgn * hstep
        vals.append(float(np.real(_solve_C(P, Xp, tp, s))))
    return (vals[0] - vals[1]) / (2 * hstep)


def adjoint_general(P, u, lam):
    """General-objective adjoint term of PAPER.md Eq. 6 with df/dp = 0 (reading c3):
    -lambda^T (dK/dp) u, where K^T lambda = dg/du (Eq. 5) is solved by the caller.
    Returns (d[3, n_nodes] for coordinates, d[n_quads] for thickness, d[n_elems] for E),
    element contributions summed in ascending element order."""
    nn = len(P["x"])
    nb, nq = A.n_beams(P), A.n_quads(P)
    X = A.coords(P)
    dX = np.zeros((3, nn))
    dt = np.zeros(nq)
    dE = np.zeros(nb + nq)
    for e in range(nb + nq):
        nodes = A.element_nodes(P, e)
        dofs = A.element_dofs(nodes)
        ue, le = u[dofs], lam[dofs]
        for il, n in enumerate(nodes):
            for axis in range(3):
                dX[axis, n] += -float(le @ element_dK_dcoord(P, e, il, axis, X) @ ue)
        if e >= nb:
            dt[e - nb] = -float(le @ element_dK_dt(P, e, X) @ ue)
        dE[e] = -float(le @ element_dK_dE(P, e, X) @ ue)
    return dX, dt, dE


def global_complex_step_linear(P, c, kind, index):
    """d(c^T u)/dp by complex step of the full solve (the pin of adjoint_general)."""
    X = A.coords(P).astype(np.complex128)
    t = P["t"].astype(np.complex128)
    Pc = P
    if kind == "xyz":
        X[index[0], index[1]] += 1j * H_CS
    elif kind == "t":
        t[index] += 1j * H_CS
    else:
        Pc = dict(P)
        Pc["E"] = P["E"].astype(np.complex128)
        Pc["E"][index] += 1j * H_CS
        if P.get("G") is not None:
            Pc["G"] = P["G"].astype(np.complex128)
            Pc["G"][index] *= Pc["E"][index] / P["E"][index]
    nd = 6 * len(P["x"])
    K = A.dense_from_dok(A.assemble_dok(Pc, X, t), nd, dtype=np.complex128)
    fixed = A.fixed_dofs(P)
    Kbc, fbc = A.apply_supports_dense(K, P["f"].astype(np.complex128), fixed)
    free = np.nonzero(~fixed)[0]
    u = np.zeros(nd, dtype=np.complex128)
    u[free] = S.solve_dense_lu(Kbc[np.ix_(free, free)], fbc[free])
    return float(np.imag(np.dot(c, u)) / H_CS)
