"""Oracle: linear solves K u = f (test infrastructure only).

PAPER.md:71-74 (Eq. 1, K u = f) and :83-96 (Eqs. 2-3, Lagrange-multiplier
supports) define the system; PAPER.md:118-134 lists the paper's direct
solvers.  BASELINE.json north_star fixes the oracle: "dense Cholesky for small
cases and CG for large ones".  The CG here is the textbook Jacobi-PCG of
SURVEY.md §8(c) C5 (reading c10):

    x0 = 0, r0 = f, z = D^-1 r, p = z;
    alpha = r.z / p.Kp;  x += alpha p;  r -= alpha Kp;
    stop when |r|_2 <= rtol |f|_2;
    beta = r_new.z_new / r_old.z_old;  p = z + beta p.

The node-block variant (reading c19, `sso_options.precond = 1`) is
the same algorithm with M = blockdiag(K_nn), the 6x6 diagonal block of every
node of K_bc (a Jacobi preconditioner over the node DOF blocks): z = M^-1 r
by a 6x6 solve per node.

Pins: tests/test_oracle_solve.py — Cholesky u equals the paper's Lagrange
augmented LU u (library special case); PCG u equals Cholesky u; true
residuals; Lanczos Ritz bounds bracket the exact extreme eigenvalues of the
Jacobi-scaled matrix on small cases.  Block PCG: u equals Cholesky u; on a
block-diagonal K it converges in one iteration (M = K); when every diagonal
block of K is itself diagonal its iterates are those of the point PCG.
"""
from __future__ import annotations

import numpy as np
import scipy.linalg as sla


def solve_dense_cholesky(K, f, fixed):
    """u on free DOFs from a dense Cholesky of K_ff; u = 0 at constrained DOFs."""
    free = np.nonzero(~fixed)[0]
    Kff = K[np.ix_(free, free)]
    c = sla.cho_factor(Kff, lower=True)
    u = np.zeros(K.shape[0], dtype=np.result_type(K, f))
    u[free] = sla.cho_solve(c, f[free])
    return u


def solve_lagrange(Kaug, faug, ndof):
    """Dense LU of the paper's augmented system (Eq. 2); returns the first ndof rows."""
    uaug = np.linalg.solve(Kaug, faug)
    return uaug[:ndof]


def solve_dense_lu(K, f):
    """Plain dense LU (used with complex-step perturbed matrices)."""
    return np.linalg.solve(K, f)


def pcg(K, f, dinv, rtol=1e-12, max_iter=100000):
    """Textbook Jacobi-PCG (see module docstring).  K: any object with K @ v
    (e.g. a scipy CSR matrix).  Returns (x, info) with info = dict(iters,
    rel_res, true_rel_res, alphas, betas)."""
    x = np.zeros_like(f)
    r = f.copy()
    z = dinv * r
    p = z.copy()
    rz = float(r @ z)
    fnorm = float(np.sqrt(f @ f))
    alphas, betas = [], []
    it = 0
    rnorm = fnorm
    if fnorm == 0.0:
        return x, dict(iters=0, rel_res=0.0, true_rel_res=0.0, alphas=[], betas=[])
    while it < max_iter:
        q = K @ p
        pq = float(p @ q)
        if pq <= 0.0:
            raise ArithmeticError("p^T K p <= 0: matrix not SPD")
        alpha = rz / pq
        x = x + alpha * p
        r = r - alpha * q
        it += 1
        alphas.append(alpha)
        rnorm = float(np.sqrt(r @ r))
        if rnorm <= rtol * fnorm:
            break
        z = dinv * r
        rz_new = float(r @ z)
        beta = rz_new / rz
        betas.append(beta)
        rz = rz_new
        p = z + beta * p
    true_r = f - K @ x
    return x, dict(iters=it, rel_res=rnorm / fnorm,
                   true_rel_res=float(np.sqrt(true_r @ true_r)) / fnorm,
                   alphas=alphas, betas=betas)


def node_blocks(K, ndof):
    """The 6x6 diagonal block of every node of K (dense or scipy sparse): [n][6][6]."""
    n = ndof // 6
    B = np.zeros((n, 6, 6))
    Kc = K.tocsr() if hasattr(K, "tocsr") else None
    for i in range(n):
        sl = slice(6 * i, 6 * i + 6)
        B[i] = Kc[sl, sl].toarray() if Kc is not None else K[sl, sl]
    return B


def pcg_block(K, f, rtol=1e-12, max_iter=100000):
    """Textbook node-block Jacobi PCG: the loop of pcg() with z = M^-1 r,
    M = blockdiag(K_nn) (reading c19).  Returns (x, info) like pcg()."""
    nd = f.shape[0]
    B = node_blocks(K, nd)

    def apply_Minv(r):
        z = np.empty_like(r)
        for i in range(nd // 6):
            z[6 * i:6 * i + 6] = np.linalg.solve(B[i], r[6 * i:6 * i + 6])
        return z

    x = np.zeros_like(f)
    r = f.copy()
    z = apply_Minv(r)
    p = z.copy()
    rz = float(r @ z)
    fnorm = float(np.sqrt(f @ f))
    it = 0
    rnorm = fnorm
    if fnorm == 0.0:
        return x, dict(iters=0, rel_res=0.0, true_rel_res=0.0)
    while it < max_iter:
        q = K @ p
        pq = float(p @ q)
        if pq <= 0.0:
            raise ArithmeticError("p^T K p <= 0: matrix not SPD")
        alpha = rz / pq
        x = x + alpha * p
        r = r - alpha * q
        it += 1
        rnorm = float(np.sqrt(r @ r))
        if rnorm <= rtol * fnorm:
            break
        z = apply_Minv(r)
        rz_new = float(r @ z)
        beta = rz_new / rz
        rz = rz_new
        p = z + beta * p
    true_r = f - K @ x
    return x, dict(iters=it, rel_res=rnorm / fnorm,
                   true_rel_res=float(np.sqrt(true_r @ true_r)) / fnorm)


def lanczos_ritz(alphas, betas):
    """Extreme Ritz values of D^-1 K from the CG coefficients: the Lanczos
    tridiagonal T has T[k,k] = 1/alpha_k + beta_{k-1}/alpha_{k-1},
    T[k,k+1] = sqrt(beta_k)/alpha_k (standard CG-Lanczos relation)."""
    m = len(alphas)
    if m == 0:
        return None, None
    T = np.zeros((m, m))
    for k in range(m):
        T[k, k] = 1.0 / alphas[k]
        if k > 0:
            T[k, k] += betas[k - 1] / alphas[k - 1]
        if k + 1 < m and k < len(betas):
            T[k, k + 1] = T[k + 1, k] = np.sqrt(betas[k]) / alphas[k]
    ev = np.linalg.eigvalsh(T)
    return float(ev[0]), float(ev[-1])
