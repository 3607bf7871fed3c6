"""Pins for oracle/solve.py (SURVEY.md §8(c) C5, C10 'Solve').

  * the dense-Cholesky u (elimination) equals the u of the paper's own
    Lagrange-multiplier system (Eq. 2-3) solved by dense LU;
  * the textbook Jacobi-PCG u equals the Cholesky u;
  * the Lanczos Ritz values bracket inside the true spectrum of D^-1/2 K D^-1/2;
  * node-block Jacobi PCG (reading c19): u equals the Cholesky u; one iteration
    on a block-diagonal K (M = K exactly); the point PCG's iterates when every
    diagonal block is diagonal.
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


def test_block_pcg_equals_cholesky_C2():
    P = W.config2()
    u_c, Kb, fb = Gd.evaluate(P, "cholesky")
    nd = 6 * len(P["x"])
    K = A.dense_from_dok(A.assemble_dok(P), nd)
    Kb, fb = A.apply_supports_dense(K, P["f"], A.fixed_dofs(P))
    u_b, info = S.pcg_block(sp.csr_matrix(Kb), fb, rtol=1e-12)
    assert np.linalg.norm(u_b - u_c) <= 1e-9 * np.linalg.norm(u_c)
    assert info["true_rel_res"] < 1e-11
    # fewer iterations than point Jacobi on a shell (rotation/translation coupling in the node block)
    d = np.diag(Kb)
    _, ip = S.pcg(sp.csr_matrix(Kb), fb, 1.0 / d, rtol=1e-12)
    assert info["iters"] < ip["iters"]


def test_block_pcg_exact_on_block_diagonal():
    rng = np.random.default_rng(5)
    n = 7
    K = np.zeros((6 * n, 6 * n))
    for i in range(n):
        Q = rng.standard_normal((6, 6))
        K[6 * i:6 * i + 6, 6 * i:6 * i + 6] = Q @ Q.T + 6 * np.eye(6)
    f = rng.standard_normal(6 * n)
    x, info = S.pcg_block(K, f, rtol=1e-14)
    assert info["iters"] == 1
    assert np.linalg.norm(x - np.linalg.solve(K, f)) <= 1e-13 * np.linalg.norm(x)


def test_block_pcg_reduces_to_point_pcg():
    # SPD K whose 6x6 diagonal blocks are diagonal: M = diag(K), the same iterates
    rng = np.random.default_rng(6)
    n = 6
    Q = rng.standard_normal((6 * n, 6 * n))
    K = Q @ Q.T + 6 * n * np.eye(6 * n)
    for i in range(n):
        blk = K[6 * i:6 * i + 6, 6 * i:6 * i + 6]
        K[6 * i:6 * i + 6, 6 * i:6 * i + 6] = np.diag(np.diag(blk))
    assert np.all(np.linalg.eigvalsh(K) > 0)
    f = rng.standard_normal(6 * n)
    for it in (1, 3, 7):
        xb, ib = S.pcg_block(K, f, rtol=0.0, max_iter=it)
        xp, ipt = S.pcg(K, f, 1.0 / np.diag(K), rtol=0.0, max_iter=it)
        assert ib["iters"] == ipt["iters"] == it
        assert np.linalg.norm(xb - xp) <= 1e-12 * np.linalg.norm(xp)
