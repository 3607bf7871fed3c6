"""GPU parity of the hat filter of sensitivities (PAPER.md:280,
349; reading c16) against oracle/filter.py, through the C-ABI (sso_hat_filter)."""
import numpy as np
import pytest

import workloads as W
from oracle import filter as OF

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def sso():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a B200"
    import paper_2407_20026_b200 as m
    return m


def _mixed():
    P = W.tiny_shell(4, seed=7, L=4.0)
    P["beam_conn"] = np.array([[0, 1], [1, 2], [2, 3], [0, 5], [5, 10]], np.int32)
    nb = 5
    P["A"], P["Iy"], P["Iz"], P["J"] = (np.full(nb, 1e-3), np.full(nb, 2e-6), np.full(nb, 1e-6),
                                        np.full(nb, 2e-6))
    P["E"] = np.concatenate([np.full(nb, 210e9), P["E"]])
    P["nu"] = np.concatenate([np.full(nb, 0.3), P["nu"]])
    return P


def _close(got, ref, tol):
    scale = np.abs(ref).max()
    assert np.abs(got - ref).max() <= tol * scale, np.abs(got - ref).max() / scale


@pytest.mark.parametrize("make", [lambda: W.tiny_shell(5, seed=2, L=5.0, zamp=0.2), _mixed])
@pytest.mark.parametrize("on_elements", [False, True])
@pytest.mark.parametrize("radius", [0.5, 1.3, 2.2, 50.0])
def test_hat_filter_small(sso, make, on_elements, radius):
    P = make()
    m = sso.Model(P)
    n = len(OF.points(P, on_elements))
    rng = np.random.default_rng(11)
    v1 = rng.standard_normal(n)
    v3 = rng.standard_normal((3, n))
    _close(m.hat_filter(v1, radius, on_elements), OF.hat_filter(P, radius, v1, on_elements), 1e-13)
    _close(m.hat_filter(v3, radius, on_elements), OF.hat_filter(P, radius, v3, on_elements), 1e-13)
    v2 = v3[:2].copy()
    _close(m.hat_filter(v2, radius, on_elements), OF.hat_filter(P, radius, v2, on_elements), 1e-13)


def test_hat_filter_device_tensors_deterministic_and_set_design(sso):
    import torch
    P = W.tiny_shell(6, seed=4, L=6.0, zamp=0.5)
    m = sso.Model(P)
    n = len(P["x"])
    v = np.random.default_rng(3).standard_normal((3, n))
    vd = torch.from_numpy(v).cuda()
    a = m.hat_filter(vd, 1.7).cpu().numpy()
    b = m.hat_filter(vd, 1.7).cpu().numpy()
    assert np.array_equal(a, b)
    assert np.array_equal(a, m.hat_filter(v, 1.7))
    _close(a, OF.hat_filter(P, 1.7, v), 1e-13)
    # new coordinates: the cached cell grid must be rebuilt
    Q = dict(P, z=P["z"] * 3.0 + 0.1 * P["x"])
    m.set_design(z=Q["z"])
    _close(m.hat_filter(v, 1.7), OF.hat_filter(Q, 1.7, v), 1e-13)
    ve = np.random.default_rng(4).standard_normal(len(Q["quad_conn"]))
    _close(m.hat_filter(ve, 0.9, True), OF.hat_filter(Q, 0.9, ve, True), 1e-13)


def test_hat_filter_errors(sso):
    P = W.tiny_shell(3, seed=1)
    m = sso.Model(P)
    v = np.zeros(len(P["x"]))
    for bad in (0.0, -1.0, float("nan"), float("inf")):
        with pytest.raises(sso.SSOError):
            m.hat_filter(v, bad)
    with pytest.raises(sso.SSOError):
        m.hat_filter(np.zeros((4, len(P["x"]))), 1.0)


@pytest.mark.parametrize("n,radius,on_elements", [(60, 1.1, False), (60, 0.4, True), (408, 0.5, False)])
def test_hat_filter_large_sampled(sso, n, radius, on_elements):
    """C3 family (up to the C3b metric mesh, 167k nodes, ~1300 neighbours per point):
    sampled output points against the definition."""
    P = W.shell_config3(n, cfg=3)
    m = sso.Model(P)
    npts = len(OF.points(P, on_elements))
    v = np.random.default_rng(n).standard_normal((3, npts))
    out = m.hat_filter(v, radius, on_elements)
    rng = np.random.default_rng(1)
    rows = np.unique(np.concatenate([[0, npts - 1, npts // 2], rng.integers(0, npts, 40)]))
    ref = OF.hat_filter_rows(P, radius, v, rows, on_elements)
    _close(out[:, rows], ref, 1e-12)


@pytest.mark.parametrize("on_elements", [False, True])
def test_hat_filter_batched_designs(sso, on_elements):
    """A batch filters every design over its own (design-dependent) coordinates: each design
    equals the oracle on that design's problem; 1- and 3-component layouts."""
    B = 3
    designs = [W.config5_design(b, n=8) for b in range(B)]
    m = sso.Model(designs[0], batch=B)
    m.set_design(z=np.stack([d["z"] for d in designs]), t=np.stack([d["t"] for d in designs]))
    n = len(OF.points(designs[0], on_elements))
    rng = np.random.default_rng(5)
    radius = 2.5
    v1 = rng.standard_normal((B, n))
    v3 = rng.standard_normal((B, 3, n))
    g1 = m.hat_filter(v1, radius, on_elements)
    g3 = m.hat_filter(v3, radius, on_elements)
    for b in range(B):
        _close(g1[b], OF.hat_filter(designs[b], radius, v1[b], on_elements), 1e-13)
        _close(g3[b], OF.hat_filter(designs[b], radius, v3[b], on_elements), 1e-13)
    # the designs differ in z, so their filters differ
    assert np.abs(g1[0] - g1[1]).max() > 0 or np.array_equal(v1[0], v1[1])
