"""GPU parity of prescribed support displacements V u = b, b != 0 (SURVEY.md §8(f) row
4; Eqs. 2-3; reading c18) against oracle/prescribed.py (the paper's Lagrange
system solved by dense LU), through the C-ABI (sso_set_prescribed):

  * u within 1e-9 of the augmented-system solution, u_c = b exactly;
  * C = s f^T u within 1e-10 and dC/dX, dC/dt, dC/dE within 1e-7 (the gradient runs a
    second PCG solve for lambda = s u_hom inside sso_grad);
  * with design-dependent area loads on top;
  * switching b off restores the plain path bit-exactly; refusals (sso_grad_at, area loads
    on a batch);
  * one b per design of a batch, equal to the single-design solves.
"""
import numpy as np
import pytest

import workloads as W
from _tol import component_err
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
    # per component with the 1e-3 |b|_inf floor
    return component_err(a, b)


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
    with pytest.raises(sso.SSOError):  # a batch takes one b per design
        mb.set_prescribed(np.full(6 * len(designs[0]["x"]), np.nan))
    # prescribed + area loads on a batch is refused at the gradient
    mb.set_prescribed(np.stack([b_vec(d, 2) for d in designs]))
    mb.set_area_load(np.full(len(designs[0]["quad_conn"]), 1e3), None)
    mb.assemble()
    mb.solve(np.stack([d["f"] for d in designs]))
    with pytest.raises(sso.SSOError):
        mb.grad(0)


@pytest.mark.parametrize("s_obj", [0, 1])
def test_prescribed_batched_designs(sso, s_obj):
    """One b per design of a batch: every design equals its single-design prescribed
    solve and gradient, and design 1 the oracle's Lagrange system."""
    B = 3
    s = 1.0 if s_obj == 0 else 0.5
    designs = [W.config5_design(k, n=8) for k in range(B)]
    bs = np.stack([b_vec(d, 10 + k) for k, d in enumerate(designs)])
    mb = sso.Model(designs[0], rtol=1e-12, batch=B)
    mb.set_design(z=np.stack([d["z"] for d in designs]), t=np.stack([d["t"] for d in designs]))
    mb.set_prescribed(bs)
    mb.assemble()
    U, infos = mb.solve(np.stack([d["f"] for d in designs]))
    assert all(i["status"] == 0 for i in infos)
    C, dX, dT = mb.grad(s_obj)
    dE = mb.grad_E(s_obj)
    fixed = OA.fixed_dofs(designs[0])
    for k in range(B):
        assert np.array_equal(U[k][fixed], bs[k][fixed])
        m1 = sso.Model(designs[k], rtol=1e-12)
        m1.set_prescribed(bs[k])
        m1.assemble()
        u1, _ = m1.solve(designs[k]["f"])
        assert np.linalg.norm(U[k] - u1) <= 1e-9 * np.linalg.norm(u1)
        c1, x1, t1 = m1.grad(s_obj)
        assert C[k] == pytest.approx(c1, rel=1e-10)
        assert _rel(dX[k], x1) <= 1e-7 and _rel(dT[k], t1) <= 1e-7
        assert _rel(dE[k], m1.grad_E(s_obj)) <= 1e-7
    P1 = designs[1]
    uref = OP.solve(P1, np.where(fixed, bs[1], 0.0))
    assert np.linalg.norm(U[1] - uref) <= 1e-9 * np.linalg.norm(uref)
    rX, rT, rE = OP.gradient(P1, uref, s)
    assert C[1] == pytest.approx(OP.compliance(P1, uref, s), rel=1e-10)
    assert _rel(dX[1], rX) <= 1e-7 and _rel(dT[1], rT) <= 1e-7 and _rel(dE[1], rE) <= 1e-7
