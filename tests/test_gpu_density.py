"""GPU parity of the SIMP density design variable (PAPER.md:343-347,
Eq. 12: E_j = p_T,j^P E_*,j) against the oracle: sso_set_density forms E = rho^P E0 (and
G = rho^P G0 or the derived G) on the device, sso_grad_density returns
dC/drho = dC/dE * P rho^(P-1) E0.  The oracle side is oracle/grad.py simp_gradient on
material_gradient, pinned to a complex step through rho in tests/test_oracle_grad.py.
Tolerances as tests/test_gpu_parity.py (u 1e-9, gradients 1e-7 with a 1e-3 max floor)."""
import numpy as np
import pytest

import workloads as W
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
