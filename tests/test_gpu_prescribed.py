"""GPU parity of prescribed support displacements V u = b, b != 0 (SURVEY.md §8(f) row
4; Eqs. 2-3; reading c18) against oracle/prescribed.py (the paper's Lagrange
system solved by dense LU), through the C-ABI (sso_set_prescribed):

  * u within 1e-9 of the augmented-system solution, u_c = b exactly;
  * C = s f^T u within 1e-10 and dC/dX, dC/dt, dC/dE within 1e-7 (the gradient runs a
    second PCG solve for lambda = s u_hom inside sso_grad);
  * with design-dependent area loads on top;
  * switching b off restores the plain path bit-exactly; refusals on batch handles and
    sso_grad_at.
"""
import numpy as np
import pytest

import workloads as W
from oracle import assembly as OA, loads as OL, prescribed as OP

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def sso():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a B200"
    import paper_2407_20026_b200 as m
    return m


def mixed():
    P = W.tiny_shell(4, seed=3)
    P["beam_conn"] = np.array([[0, 6], [6, 12], [3, 9], [20, 24]], np.int32)
    nb = len(P["beam_conn"])
    P["A"], P["Iy"], P["Iz"], P["J"] = (np.full(nb, 1e-3), np.full(nb, 2e-6), np.full(nb, 1e-6),
                                        np.full(nb, 2e-6))
    P["E"] = np.concatenate([np.full(nb, 210e9), P["E"]])
    P["nu"] = np.concatenate([np.full(nb, 0.3), P["nu"]])
    return P


def b_vec(P, seed):
    rng = np.random.default_rng(seed)
    b = rng.uniform(-1e-3, 1e-3, 6 * len(P["x"]))  # free entries must be ignored
    return b


def _rel(a, b):
    return np.abs(a - b).max() / np.abs(b).max()


MAKERS = {"tiny2": lambda: W.tiny_shell(2, 0), "tiny3": lambda: W.tiny_shell(3, 2), "mixed": mixed,
          "beams": lambda: W.tiny_beam_grid(1), "C2": W.config2}


@pytest.mark.parametrize("name", list(MAKERS))
@pytest.mark.parametrize("s_obj", [0, 1])
def test_prescribed_solve_and_gradient(sso, name, s_obj):
    P = MAKERS[name]()
    s = 1.0 if s_obj == 0 else 0.5
    b = b_vec(P, 5)
    fixed = OA.fixed_dofs(P)
    m = sso.Model(P, rtol=1e-12)
    m.set_prescribed(b)
    m.assemble()
    u, info = m.solve(P["f"])
    assert info["status"] == 0
    uref = OP.solve(P, np.where(fixed, b, 0.0))
    assert np.array_equal(u[fixed], b[fixed])
    assert np.linalg.norm(u - uref) <= 1e-9 * np.linalg.norm(uref)
    C, dX, dT = m.grad(s_obj)
    assert C == pytest.approx(OP.compliance(P, uref, s), rel=1e-10)
    rX, rT, rE = OP.gradient(P, uref, s)
    assert _rel(dX, rX) <= 1e-7
    if len(rT):
        assert _rel(dT, rT) <= 1e-7
    dE = m.grad_E(s_obj)
    assert _rel(dE, rE) <= 1e-7
    # the primal survives the internal adjoint solve
    C2, dX2, _ = m.grad(s_obj)
    assert C2 == C and np.array_equal(dX2, dX)
    # off again: bit-exact with a fresh handle
    m.set_prescribed(None)
    m.assemble()
    u0, _ = m.solve(P["f"])
    m0 = sso.Model(P, rtol=1e-12)
    m0.assemble()
    u1, _ = m0.solve(P["f"])
    assert np.array_equal(u0, u1)
    assert np.array_equal(m.grad(s_obj)[1], m0.grad(s_obj)[1])


def test_prescribed_with_area_loads(sso):
    P = W.tiny_shell(3, 4)
    rng = np.random.default_rng(5)
    nq = len(P["quad_conn"])
    q, w, d = rng.uniform(1e3, 3e3, nq), rng.uniform(2e4, 3e4, nq), np.array([0.1, 0.3, -1.0])
    b = b_vec(P, 7)
    fixed = OA.fixed_dofs(P)
    s = 0.5
    m = sso.Model(P, rtol=1e-12)
    m.set_prescribed(b)
    m.set_area_load(q, w, d)
    m.assemble()
    u, _ = m.solve(P["f"])
    f = P["f"] + OL.area_load(P, q, w, d)
    uref = OP.solve(P, np.where(fixed, b, 0.0), f)
    assert np.linalg.norm(u - uref) <= 1e-9 * np.linalg.norm(uref)
    C, dX, dT = m.grad(1)
    assert C == pytest.approx(s * float(np.dot(f, uref)), rel=1e-10)
    rX, rT, _ = OP.gradient_with_loads(P, uref, q, w, d, s)
    assert _rel(dX, rX) <= 1e-7 and _rel(dT, rT) <= 1e-7


def test_prescribed_refusals(sso):
    P = W.tiny_shell(2, 0)
    m = sso.Model(P)
    m.set_prescribed(b_vec(P, 1))
    with pytest.raises(sso.SSOError):  # needs a new assembly
        m.solve(P["f"])
    m.assemble()
    m.solve(P["f"])
    with pytest.raises(sso.SSOError):
        m.grad_at(P["f"], np.zeros(6 * len(P["x"])))
    designs = [W.config5_design(k, n=6) for k in range(2)]
    mb = sso.Model(designs[0], batch=2)
    with pytest.raises(sso.SSOError):
        mb.set_prescribed(b_vec(designs[0], 2))
