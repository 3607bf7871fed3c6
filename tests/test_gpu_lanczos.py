"""GPU certification of the CG solve (include/sso.h sso_solve_info lanczos_* / err_*;
csrc/lanczos.cu).  PAPER.md:71-74 (Eq. 1) solved by CG; SURVEY.md §8(c) C5.

The device forms the extreme Ritz values of M^-1 K from the CG coefficients.  They are
pinned against the generalized eigenvalues of (K_bc, M) from LAPACK (scipy eigh on the
oracle's dense K_bc, a library routine independent of both CG runs): the Ritz values must
lie inside the spectrum (interlacing) and, after a converged solve, match its ends; and
against the oracle's own Lanczos (oracle/solve.py lanczos_ritz over its PCG coefficients).
The error estimates must bound the actual error of u against the oracle's Cholesky u.
"""
import numpy as np
import pytest
import scipy.linalg as sla

import workloads as W
from oracle import assembly as OA, grad as OG, solve as OS

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def sso():
    import paper_2407_20026_b200 as m
    return m


def _dense_bc(P):
    nd = 6 * len(P["x"])
    K = OA.dense_from_dok(OA.assemble_dok(P), nd)
    Kb, fb = OA.apply_supports_dense(K, P["f"], OA.fixed_dofs(P))
    return Kb, fb


def _M(Kb, precond):
    if precond == 0:
        return np.diag(np.diag(Kb))
    M = np.zeros_like(Kb)
    for n in range(Kb.shape[0] // 6):
        s = slice(6 * n, 6 * n + 6)
        M[s, s] = Kb[s, s]
    return M


@pytest.mark.parametrize("precond", [0, 1])
@pytest.mark.parametrize("make", [W.config2, lambda: W.tiny_shell(3, 2), W.config1])
def test_ritz_values_and_error_estimates(sso, make, precond):
    P = make()
    Kb, fb = _dense_bc(P)
    ev = sla.eigh(Kb, _M(Kb, precond), eigvals_only=True)
    lam_min, lam_max = ev[0], ev[-1]
    m = sso.Model(P, rtol=1e-12, precond=precond, device=0)
    m.assemble()
    u, info = m.solve(P["f"])
    assert info["status"] == 0 and info["lanczos_iters"] == info["iters"]
    lo, hi = info["lanczos_lmin"], info["lanczos_lmax"]
    # interlacing (up to the multisection width) and convergence to the spectrum's ends
    assert lam_min * (1 - 1e-8) <= lo <= lam_min * (1 + 1e-3), (lo, lam_min)
    assert lam_max * (1 - 1e-6) <= hi <= lam_max * (1 + 1e-8), (hi, lam_max)
    # the oracle's own Lanczos on its PCG coefficients (point Jacobi)
    if precond == 0:
        dinv = 1.0 / np.diag(Kb)
        _, oi = OS.pcg(Kb, fb, dinv, rtol=1e-12)
        olo, ohi = OS.lanczos_ritz(oi["alphas"], oi["betas"][:len(oi["alphas"]) - 1])
        assert lo == pytest.approx(olo, rel=1e-3) and hi == pytest.approx(ohi, rel=1e-6)
    # the error estimates bound the actual error of u (oracle Cholesky u)
    uref, _, _ = OG.evaluate(P)
    e = u - uref
    eK = np.sqrt(e @ Kb @ e) / np.sqrt(uref @ Kb @ uref)
    e2 = np.linalg.norm(e) / np.linalg.norm(uref)
    assert np.isfinite(info["err_energy_est"]) and np.isfinite(info["err2_est"])
    # (the estimates use the GPU's own residual: allow the oracle's rounding on top)
    assert eK <= 1.01 * info["err_energy_est"] + 1e-14, (eK, info["err_energy_est"])
    assert e2 <= 1.01 * info["err2_est"] + 1e-13, (e2, info["err2_est"])
    assert info["err2_est"] < 1e-6


def test_ritz_batched_designs(sso):
    """Every design of a batch gets its own Ritz values, equal (to the multisection width)
    to a single-design solve of that design."""
    designs = [W.config5_design(d, n=12) for d in range(3)]
    mb = sso.Model(designs[0], rtol=1e-12, batch=3, device=0)
    mb.set_design(z=np.stack([d["z"] for d in designs]), t=np.stack([d["t"] for d in designs]))
    mb.assemble()
    _, infos = mb.solve(np.stack([d["f"] for d in designs]))
    for d, ib in zip(designs, infos):
        m1 = sso.Model(d, rtol=1e-12, device=0)
        m1.assemble()
        _, i1 = m1.solve(d["f"])
        assert ib["lanczos_lmax"] == pytest.approx(i1["lanczos_lmax"], rel=1e-7)
        assert ib["lanczos_lmin"] == pytest.approx(i1["lanczos_lmin"], rel=1e-5)
