"""GPU parity of the design-dependent area loads (PAPER.md
Eq. 6 with df/dp != 0; reading c17) against oracle/loads.py, through the C-ABI
(sso_set_area_load + sso_solve / sso_grad / sso_adjoint_solve / sso_grad_adjoint):

  * u within 1e-9 of the oracle (Cholesky) with f = nodal loads + area load, and with
    the area load alone (f = NULL);
  * dC/dX, dC/dt = s (2 u^T df/dp - u^T dK/dp u) within 1e-7 of the oracle;
  * general adjoint -lambda^T (dK/dp u - df/dp), with the adjoint solve ignoring the load;
  * partitioned strips and batched designs equal the single-strip handle;
  * switching the load off restores the fixed-load results bit-exactly.
"""
import numpy as np
import pytest

import workloads as W
from _tol import component_err
from oracle import grad as OG, loads as OL

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


def load_case(P, seed=0):
    rng = np.random.default_rng(seed)
    nq = len(P["quad_conn"])
    return rng.uniform(1e3, 3e3, nq), rng.uniform(2e4, 3e4, nq), np.array([0.2, -0.1, -1.0])


def _rel(a, b):
    # per component with the 1e-3 |b|_inf floor
    return component_err(a, b)


MAKERS = {"tiny2": lambda: W.tiny_shell(2, 0), "tiny3": lambda: W.tiny_shell(3, 5), "mixed": mixed,
          "C2": W.config2}


@pytest.mark.parametrize("name", list(MAKERS))
@pytest.mark.parametrize("s_obj", [0, 1])
def test_area_load_solve_and_gradient(sso, name, s_obj):
    P = MAKERS[name]()
    q, w, d = load_case(P, 1)
    s = 1.0 if s_obj == 0 else 0.5
    m = sso.Model(P, rtol=1e-12)
    m.assemble()
    m.set_area_load(q, w, d)
    u, info = m.solve(P["f"])
    assert info["status"] == 0
    uref, fref = OL.evaluate(P, q, w, d)
    assert np.linalg.norm(u - uref) <= 1e-9 * np.linalg.norm(uref)
    C, dX, dT = m.grad(s_obj)
    assert C == pytest.approx(s * float(np.dot(fref, uref)), rel=1e-10)
    rX, rT = OL.compliance_gradient(P, uref, q, w, d, s)
    assert _rel(dX, rX) <= 1e-7
    assert _rel(dT, rT) <= 1e-7
    # the area load alone (f = NULL)
    u0, _ = m.solve(None)
    uref0, _ = OL.evaluate(dict(P, f=np.zeros_like(P["f"])), q, w, d)
    assert np.linalg.norm(u0 - uref0) <= 1e-9 * np.linalg.norm(uref0)
    # switched off: the fixed-load path, bit-exact against a fresh handle
    m.set_area_load(None, None)
    uf, _ = m.solve(P["f"])
    Cf, dXf, dTf = m.grad(s_obj)
    m2 = sso.Model(P, rtol=1e-12)
    m2.assemble()
    u2, _ = m2.solve(P["f"])
    C2, dX2, dT2 = m2.grad(s_obj)
    assert np.array_equal(uf, u2) and np.array_equal(dXf, dX2) and Cf == C2


@pytest.mark.parametrize("make", [lambda: W.tiny_shell(3, 4), mixed])
def test_area_load_general_adjoint(sso, make):
    P = make()
    q, w, d = load_case(P, 2)
    m = sso.Model(P, rtol=1e-12)
    m.assemble()
    m.set_area_load(q, w, d)
    u, _ = m.solve(P["f"])
    uref, fref = OL.evaluate(P, q, w, d)
    from oracle import assembly as OA
    fixed = OA.fixed_dofs(P)
    c = np.random.default_rng(6).standard_normal(m.ndof)
    c[fixed] = 0.0
    lam, info = m.adjoint_solve(c)
    _, Kb, _ = OG.evaluate(P)
    free = np.nonzero(~fixed)[0]
    lref = np.zeros_like(uref)
    lref[free] = np.linalg.solve(Kb[np.ix_(free, free)], c[free])
    assert np.linalg.norm(lam - lref) <= 1e-9 * np.linalg.norm(lref)
    dX, dT, dE = m.grad_adjoint(lref)
    rX, rT, rE = OG.adjoint_general(P, uref, lref)
    lX, lT = OL.load_gradient_term(P, lref, q, w, d)
    assert _rel(dX, rX + lX) <= 1e-7
    assert _rel(dT, rT + lT) <= 1e-7
    assert _rel(dE, rE) <= 1e-7


@pytest.mark.parametrize("nparts", [2, 3])
def test_area_load_partitioned_matches_single(sso, nparts):
    P = W.config2()
    q, w, d = load_case(P, 3)
    m1 = sso.Model(P, rtol=1e-12, storage=1)
    m1.assemble()
    m1.set_area_load(q, w, d)
    u1, _ = m1.solve(None)
    C1, dX1, dT1 = m1.grad()
    mp = sso.Model(P, rtol=1e-12, n_parts=nparts)
    mp.assemble()
    mp.set_area_load(q, w, d)
    up, _ = mp.solve(None)
    Cp, dXp, dTp = mp.grad()
    assert np.linalg.norm(up - u1) <= 1e-9 * np.linalg.norm(u1)
    assert Cp == pytest.approx(C1, rel=1e-10)
    assert _rel(dXp, dX1) <= 1e-7 and _rel(dTp, dT1) <= 1e-7


def test_area_load_batched_designs(sso):
    B = 3
    designs = [W.config5_design(b, n=12) for b in range(B)]
    P0 = designs[0]
    q, w, d = load_case(P0, 4)
    mb = sso.Model(P0, rtol=1e-12, batch=B)
    mb.set_design(z=np.stack([x["z"] for x in designs]), t=np.stack([x["t"] for x in designs]))
    mb.assemble()
    mb.set_area_load(q, w, d)
    F = np.stack([x["f"] for x in designs])
    U, infos = mb.solve(F)
    Cb, dXb, dTb = mb.grad()
    for b, x in enumerate(designs):
        m1 = sso.Model(x, rtol=1e-12)
        m1.assemble()
        m1.set_area_load(q, w, d)
        u1, _ = m1.solve(x["f"])
        assert np.linalg.norm(U[b] - u1) <= 1e-9 * np.linalg.norm(u1)
        C1, dX1, dT1 = m1.grad()
        assert Cb[b] == pytest.approx(C1, rel=1e-10)
        assert _rel(dXb[b], dX1) <= 1e-7 and _rel(dTb[b], dT1) <= 1e-7
    uref, _ = OL.evaluate(designs[1], q, w, d)
    assert np.linalg.norm(U[1] - uref) <= 1e-9 * np.linalg.norm(uref)
