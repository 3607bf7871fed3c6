"""Pin of reading c21: the single-reduction (Chronopoulos-Gear) rearrangement that
the partitioned handles run (csrc/cg_sr.cu) produces the iterates of the textbook Jacobi-PCG of
reading c10 (oracle/solve.py pcg).  Written out here in numpy from the recurrences in the
cg_sr.cu header -- alpha_i = gamma_i / (delta_i - beta_i gamma_i / alpha_{i-1}), s = K p
carried by s = w + beta s -- and compared with the oracle's loop on small SPD systems: equal
iterates to rounding, the same iteration count, and (alpha, beta) pairs that give the oracle's
Lanczos Ritz values."""
import numpy as np
import pytest

import workloads as W
from oracle import assembly as OA, grad as OG, solve as OS


def single_reduction_pcg(K, f, dinv, rtol, max_iter=100000):
    x = np.zeros_like(f)
    r = f.copy()
    u = dinv * r
    p = np.zeros_like(f)
    s = np.zeros_like(f)
    ff = float(f @ f)
    alpha_prev = gamma_prev = None
    alphas, betas = [], []
    it = 0
    while True:
        w = K @ u
        gamma, delta, rr = float(r @ u), float(u @ w), float(r @ r)
        if rr <= rtol * rtol * ff or it >= max_iter:
            break
        if it == 0:
            beta, den = 0.0, delta
        else:
            beta = gamma / gamma_prev
            den = delta - beta * gamma / alpha_prev
            betas.append(beta)
        alpha = gamma / den
        alphas.append(alpha)
        p = u + beta * p
        s = w + beta * s
        x = x + alpha * p
        r = r - alpha * s
        u = dinv * r
        alpha_prev, gamma_prev = alpha, gamma
        it += 1
    return x, it, alphas, betas


@pytest.mark.parametrize("make", [W.config2, lambda: W.tiny_shell(3, 2), W.config1,
                                  lambda: W.shell_config3(12, cfg=4, supports="c4")])
def test_single_reduction_equals_textbook_pcg(make):
    P = make()
    nd = 6 * len(P["x"])
    K = OA.dense_from_dok(OA.assemble_dok(P), nd)
    Kb, fb = OA.apply_supports_dense(K, P["f"], OA.fixed_dofs(P))
    dinv = 1.0 / np.diag(Kb)
    x_ref, info = OS.pcg(Kb, fb, dinv, rtol=1e-10)
    x, it, alphas, betas = single_reduction_pcg(Kb, fb, dinv, 1e-10)
    assert abs(it - info["iters"]) <= max(3, 0.02 * info["iters"])
    assert np.linalg.norm(x - x_ref) <= 1e-8 * np.linalg.norm(x_ref)
    # the coefficients are the textbook ones: the same Lanczos tridiagonal
    n = min(len(alphas), len(info["alphas"])) - 1
    assert np.allclose(alphas[:20], info["alphas"][:20], rtol=1e-9)
    lo, hi = OS.lanczos_ritz(alphas[:n], betas[:n - 1])
    lo_r, hi_r = OS.lanczos_ritz(info["alphas"][:n], info["betas"][:n - 1])
    assert hi == pytest.approx(hi_r, rel=1e-8) and lo == pytest.approx(lo_r, rel=1e-4)
    u_c, _, _ = OG.evaluate(P)
    assert np.linalg.norm(x - u_c) <= 1e-8 * np.linalg.norm(u_c)
