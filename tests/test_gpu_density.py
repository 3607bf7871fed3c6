"""GPU parity of the SIMP density design variable (PAPER.md:343-347,
Eq. 12: E_j = p_T,j^P E_*,j) against the oracle: sso_set_density forms E = rho^P E0 (and
G = rho^P G0 or the derived G) on the device, sso_grad_density returns
dC/drho = dC/dE * P rho^(P-1) E0.  The oracle side is oracle/grad.py simp_gradient on
material_gradient, pinned to a complex step through rho in tests/test_oracle_grad.py.
Tolerances as tests/test_gpu_parity.py (u 1e-9, gradients 1e-7 with a 1e-3 max floor).
Also the batched general-objective adjoint."""
import numpy as np
import pytest

import workloads as W
from _tol import assert_components
from oracle import grad as OG

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def sso():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a B200"
    import paper_2407_20026_b200 as m
    return m


@pytest.mark.parametrize("penal", [3.0, 7.0])
@pytest.mark.parametrize("make", [W.config2, W.config1, lambda: W.tiny_beam_grid(2)])
def test_simp_density_against_oracle(sso, make, penal):
    P = make()
    ne = len(P["E"])
    rho = np.random.default_rng(11).uniform(0.3, 1.0, ne)
    E0 = np.asarray(P["E"], np.float64).copy()
    G0 = None if P.get("G") is None else np.asarray(P["G"], np.float64).copy()
    m = sso.Model(P, rtol=1e-12)
    m.set_density(rho, penal, E0, G0)
    m.assemble()
    u, info = m.solve(P["f"])
    assert info["status"] == 0
    f = rho ** penal
    Q = dict(P, E=f * E0, G=None if G0 is None else f * G0)
    uref, _, _ = OG.evaluate(Q)
    assert np.linalg.norm(u - uref) <= 1e-9 * np.linalg.norm(uref)
    g = m.grad_density()
    ref = OG.simp_gradient(OG.material_gradient(Q, uref, 1.0), rho, E0, penal)
    floor = 1e-3 * np.abs(ref).max()
    assert np.all(np.abs(g - ref) <= 1e-7 * np.maximum(np.abs(ref), floor))
    # strain energy objective: half of it
    g2 = m.grad_density(sso.OBJ_STRAIN_ENERGY)
    assert np.allclose(g2, 0.5 * g, rtol=1e-12, atol=0.0)


def test_simp_density_errors_and_material_reset(sso):
    P = W.config2()
    ne = len(P["E"])
    m = sso.Model(P, rtol=1e-12)
    with pytest.raises(sso.SSOError):
        m.grad_density()                      # no density set
    with pytest.raises(sso.SSOError):
        m.set_density(np.full(ne, 1.5), 3.0, P["E"])   # rho > 1
    with pytest.raises(sso.SSOError):
        m.set_density(np.full(ne, 0.5), 0.5, P["E"])   # P < 1
    m.set_density(np.full(ne, 0.5), 3.0, P["E"])
    m.set_material(P["E"])                    # back to the given moduli: density mode ends
    m.assemble()
    u, _ = m.solve(P["f"])
    uref, _, _ = OG.evaluate(P)
    assert np.linalg.norm(u - uref) <= 1e-9 * np.linalg.norm(uref)
    with pytest.raises(sso.SSOError):
        m.grad_density()


@pytest.mark.parametrize("precond", [0, 1])
def test_batched_general_adjoint(sso, precond):
    """SURVEY.md §8(f) row 2 "a second (batched) PCG with rhs dg/du": a batch of designs
    solves its adjoints together and each design's lambda and -lambda^T (dK/dp) u equal the
    single-design ones (and, for one design, the oracle's)."""
    from oracle import assembly as OA
    B = 4
    designs = [W.config5_design(b, n=10) for b in range(B)]
    Z = np.stack([d["z"] for d in designs])
    T = np.stack([d["t"] for d in designs])
    F = np.stack([d["f"] for d in designs])
    fixed = OA.fixed_dofs(designs[0])
    rng = np.random.default_rng(21)
    Cg = rng.standard_normal((B, 6 * len(designs[0]["x"])))
    Cg[:, fixed] = 0.0
    mb = sso.Model(designs[0], rtol=1e-12, batch=B, precond=precond)
    mb.set_design(z=Z, t=T)
    mb.assemble()
    U, _ = mb.solve(F)
    Lam, infos = mb.adjoint_solve(Cg)
    assert all(i["status"] == 0 for i in infos)
    dX, dT, dE = mb.grad_adjoint(Lam)
    for b in (0, 3):
        m1 = sso.Model(designs[b], rtol=1e-12, precond=precond)
        m1.assemble()
        u1, _ = m1.solve(designs[b]["f"])
        l1, _ = m1.adjoint_solve(Cg[b])
        assert np.linalg.norm(U[b] - u1) <= 1e-9 * np.linalg.norm(u1)
        assert np.linalg.norm(Lam[b] - l1) <= 1e-9 * np.linalg.norm(l1)
        x1, t1, e1 = m1.grad_adjoint(l1)
        for got, ref in ((dX[b], x1), (dT[b], t1), (dE[b], e1)):
            fl = 1e-3 * np.abs(ref).max()
            assert np.all(np.abs(got - ref) <= 1e-7 * np.maximum(np.abs(ref), fl))
    # design 2 against the oracle
    P2 = designs[2]
    uref, _, _ = OG.evaluate(P2)
    rX, rT, rE = OG.adjoint_general(P2, uref, Lam[2])
    for got, ref in ((dX[2], rX), (dT[2], rT), (dE[2], rE)):
        assert_components(got, ref, 1e-7, "batched general adjoint vs oracle")
