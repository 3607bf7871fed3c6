"""Oracle: prescribed non-zero support displacements V u = b (test infrastructure
only).

PAPER.md:83-96 (Eqs. 2-3): the paper imposes supports with Lagrange multipliers,
K_aug = [[K, V^T], [V, 0]], f_aug = (f; b), V u = b, and keeps b general.  The
oracle solves exactly that augmented system (dense LU, oracle/solve.py
solve_lagrange); the GPU path eliminates instead (lifting, reading c18).

Objective (reading c18): C = s f^T u with u the full displacement (u_c = b at the
constrained DOFs).  Eq. 5-6 on the augmented system, with V and b independent of
the design p:

    K_aug lambda_aug = (s f; 0)    =>   lambda = s u_hom, u_hom the solution of the
                                         same loads with b = 0 (lambda_c = 0)
    dC/dp = -lambda^T (dK/dp) u                                     (f fixed)

(with b = 0, u_hom = u and this is the self-adjoint -s u^T dK/dp u of grad.py).
Pins (tests/test_oracle_prescribed.py): the global complex step of the full
augmented solve; the b = 0 special case; a rigid-body translation prescribed at
every support of a free-standing structure moves it rigidly (u = b everywhere,
K u = 0, C = s f^T u).
"""
from __future__ import annotations

import numpy as np

from . import assembly as A
from . import grad as Gd
from . import solve as S


def constrained_values(P, b_full):
    """b for the constrained DOFs (ascending DOF order) from a full [6 n] vector."""
    return b_full[np.nonzero(A.fixed_dofs(P))[0]]


def solve(P, b_full, f=None, X=None, t=None):
    """u from the paper's augmented system (Eq. 2) with V u = b (Eq. 3)."""
    nd = 6 * len(P["x"])
    if f is None:
        f = P["f"]
    dok = A.assemble_dok(P, X, t)
    cplx = (X is not None and np.iscomplexobj(X)) or (t is not None and np.iscomplexobj(t))
    K = A.dense_from_dok(dok, nd, dtype=np.complex128 if cplx else np.float64)
    fixed = A.fixed_dofs(P)
    Kaug, faug = A.lagrange_system(K, f, fixed, constrained_values(P, b_full))
    return S.solve_lagrange(Kaug, faug, nd)


def compliance(P, u, s=1.0):
    return s * float(np.real(np.dot(P["f"], u)))


def gradient(P, u, s=1.0):
    """dC/dX [3, n], dC/dt [n_quads], dC/dE [n_elems] = -lambda^T dK/dp u, lambda = s u_hom."""
    u_hom = solve(P, np.zeros(6 * len(P["x"])))
    dX, dt, dE = Gd.adjoint_general(P, u, s * u_hom)
    return dX, dt, dE


def gradient_with_loads(P, u, q, w, d, s=1.0):
    """With design-dependent area loads as well (oracle/loads.py, reading c17), f the total
    load: dC/dp = -lambda^T dK/dp u + (lambda + s u)^T df/dp, lambda = s u_hom(f)."""
    from . import loads as L
    f = P["f"] + L.area_load(P, q, w, d)
    u_hom = solve(P, np.zeros(6 * len(P["x"])), f)
    lam = s * u_hom
    dX, dt, dE = Gd.adjoint_general(P, u, lam)
    lX, lt = L.load_gradient_term(P, lam + s * u, q, w, d)
    return dX + lX, dt + lt, dE


def global_complex_step(P, b_full, kind, index, s=1.0, load=None):
    """dC/dp by complex step of the augmented solve (b fixed; f fixed, or recomputed
    from the area load model when load = (q, w, d))."""
    X = A.coords(P).astype(np.complex128)
    t = P["t"].astype(np.complex128)
    h = Gd.H_CS
    if kind == "xyz":
        X[index[0], index[1]] += 1j * h
    else:
        t[index] += 1j * h
    f = P["f"].astype(np.complex128)
    if load is not None:
        from . import loads as L
        f = f + L.area_load(P, *load, X, t)
    u = solve(P, b_full, f, X, t)
    return float(np.imag(s * np.dot(f, u)) / h)
