"""Pins for oracle/solve.py (SURVEY.md §8(c) C5, C10 'Solve').

  * the dense-Cholesky u (elimination) equals the u of the paper's own
    Lagrange-multiplier system (Eq. 2-3) solved by dense LU;
  * the textbook Jacobi-PCG u equals the Cholesky u;
  * the Lanczos Ritz values bracket inside the true spectrum of D^-1/2 K D^-1/2.
"""
import numpy as np
import pytest
import scipy.sparse as sp

import workloads as W
from oracle import assembly as A, grad as Gd, solve as S


@pytest.mark.parametrize("make", [lambda: W.tiny_shell(2, 0), lambda: W.tiny_shell(3, 1),
                                  lambda: W.tiny_beam_grid(0), W.config1,
                                  lambda: W.tiny_shell(3, 2, supports="edge")])
def test_cholesky_equals_lagrange(make):
    P = make()
    nd = 6 * len(P["x"])
    K = A.dense_from_dok(A.assemble_dok(P), nd)
    fixed = A.fixed_dofs(P)
    Kb, fb = A.apply_supports_dense(K, P["f"], fixed)
    u = S.solve_dense_cholesky(Kb, fb, fixed)
    Kaug, faug = A.lagrange_system(K, P["f"], fixed)
    ul = S.solve_lagrange(Kaug, faug, nd)
    assert np.linalg.norm(u - ul) <= 1e-10 * np.linalg.norm(u)
    # residual of the eliminated system
    assert np.linalg.norm(Kb @ u - fb) <= 1e-9 * np.linalg.norm(fb)


def test_pcg_equals_cholesky_C2():
    P = W.config2()
    u_c, Kb, fb = Gd.evaluate(P, "cholesky")
    u_p, Kc, _ = Gd.evaluate(P, "pcg", rtol=1e-12)
    assert np.linalg.norm(u_p - u_c) <= 1e-9 * np.linalg.norm(u_c)


def test_lanczos_bounds():
    P = W.tiny_shell(3, 4)
    nd = 6 * len(P["x"])
    K = A.dense_from_dok(A.assemble_dok(P), nd)
    fixed = A.fixed_dofs(P)
    Kb, fb = A.apply_supports_dense(K, P["f"], fixed)
    d = np.diag(Kb)
    x, info = S.pcg(sp.csr_matrix(Kb), fb, 1.0 / d, rtol=1e-14, max_iter=40)
    lmin, lmax = S.lanczos_ritz(info["alphas"], info["betas"][:len(info["alphas"]) - 1])
    ev = np.linalg.eigvalsh(Kb / np.sqrt(np.outer(d, d)))
    assert ev[0] * (1 - 1e-8) <= lmin and lmax <= ev[-1] * (1 + 1e-8)
    assert lmax >= 0.5 * ev[-1]
