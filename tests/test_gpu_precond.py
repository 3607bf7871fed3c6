"""GPU parity of the NEXT-row paths with the node-block Jacobi
preconditioner (sso_options.precond = 1, reading c19) against the oracle:
the preconditioner changes the CG iterates, never the solutions.

  * general-objective adjoint solve K lambda = c and -lambda^T dK/dp u;
  * design-dependent area loads (reading c17) and their gradient;
  * prescribed supports b != 0 (reading c18, lifting + internal second solve);
  * SIMP material gradient dC/dE.
Tolerances as in tests/test_gpu_parity.py (u 1e-9, C 1e-10, gradients 1e-7 per component
with the 1e-3 floor).
"""
import numpy as np
import pytest

import workloads as W
from _tol import component_err
from oracle import assembly as OA, grad as OG, loads as OL, prescribed as OP

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def sso():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a B200"
    import paper_2407_20026_b200 as m
    return m


def _rel(a, b):
    # per component with the 1e-3 |b|_inf floor
    return component_err(a, b)


@pytest.mark.parametrize("storage", [1, 3])
def test_block_jacobi_adjoint_and_material(sso, storage):
    P = W.config2()
    m = sso.Model(P, rtol=1e-12, precond=1, storage=storage)
    m.assemble()
    u, info = m.solve(P["f"])
    assert info["status"] == 0
    uref, Kb, _ = OG.evaluate(P)
    assert np.linalg.norm(u - uref) <= 1e-9 * np.linalg.norm(uref)
    fixed = OA.fixed_dofs(P)
    c = np.random.default_rng(8).standard_normal(m.ndof)
    c[fixed] = 0.0
    lam, li = m.adjoint_solve(c)
    assert li["status"] == 0
    free = np.nonzero(~fixed)[0]
    lref = np.zeros_like(uref)
    lref[free] = np.linalg.solve(Kb[np.ix_(free, free)], c[free])
    assert np.linalg.norm(lam - lref) <= 1e-9 * np.linalg.norm(lref)
    g = m.grad_E()
    ref = OG.material_gradient(P, uref, 1.0)
    fl = 1e-3 * np.abs(ref).max()
    assert np.all(np.abs(g - ref) <= 1e-7 * np.maximum(np.abs(ref), fl))


def test_block_jacobi_area_loads(sso):
    P = W.tiny_shell(3, 5)
    rng = np.random.default_rng(1)
    nq = len(P["quad_conn"])
    q, w, d = rng.uniform(1e3, 3e3, nq), rng.uniform(2e4, 3e4, nq), np.array([0.2, -0.1, -1.0])
    m = sso.Model(P, rtol=1e-12, precond=1)
    m.assemble()
    m.set_area_load(q, w, d)
    u, info = m.solve(P["f"])
    assert info["status"] == 0
    uref, fref = OL.evaluate(P, q, w, d)
    assert np.linalg.norm(u - uref) <= 1e-9 * np.linalg.norm(uref)
    C, dX, dT = m.grad(0)
    assert C == pytest.approx(float(np.dot(fref, uref)), rel=1e-10)
    rX, rT = OL.compliance_gradient(P, uref, q, w, d, 1.0)
    assert _rel(dX, rX) <= 1e-7 and _rel(dT, rT) <= 1e-7


def test_block_jacobi_prescribed(sso):
    P = W.config2()
    b = np.random.default_rng(5).uniform(-1e-3, 1e-3, 6 * len(P["x"]))
    fixed = OA.fixed_dofs(P)
    m = sso.Model(P, rtol=1e-12, precond=1)
    m.set_prescribed(b)
    m.assemble()
    u, info = m.solve(P["f"])
    assert info["status"] == 0
    uref = OP.solve(P, np.where(fixed, b, 0.0))
    assert np.array_equal(u[fixed], b[fixed])
    assert np.linalg.norm(u - uref) <= 1e-9 * np.linalg.norm(uref)
    C, dX, dT = m.grad(0)
    assert C == pytest.approx(OP.compliance(P, uref, 1.0), rel=1e-10)
    rX, rT, rE = OP.gradient(P, uref, 1.0)
    assert _rel(dX, rX) <= 1e-7 and _rel(dT, rT) <= 1e-7
