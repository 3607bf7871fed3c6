"""Pins for oracle/loads.py (design-dependent area loads, SURVEY.md §8(f) row 4;
PAPER.md Eq. 6 with df/dp != 0; reading c17)."""
import numpy as np
import pytest

import workloads as W
from oracle import grad as Gd, loads as L


def _load_case(P, seed=0):
    rng = np.random.default_rng(seed)
    nq = len(P["quad_conn"])
    return rng.uniform(1e3, 3e3, nq), rng.uniform(2e4, 3e4, nq), np.array([0.2, -0.1, -1.0])


def test_flat_rectangle_total_load_closed_form():
    n, Lx = 4, 3.0
    x, y = W.grid_nodes(n, Lx)
    conn = W.grid_quads(n)
    nq = len(conn)
    P = W._problem("flat", x, y, np.zeros_like(x), quad_conn=conn, t=np.full(nq, 0.2),
                   E=np.full(nq, 30e9), nu=np.full(nq, 0.2), sup_node=[0], sup_mask=[W.CLAMPED],
                   f=np.zeros(6 * len(x)))
    d = np.array([0.0, 0.0, -1.0])
    f = L.area_load(P, np.full(nq, 2e3), np.full(nq, 24e3), d)
    assert f[2::6].sum() == pytest.approx(-(2e3 + 24e3 * 0.2) * Lx * Lx, rel=1e-14)
    assert np.all(f[0::6] == 0) and np.all(f[3::6] == 0)


def test_matches_generator_lumping():
    P = W.shell_config3(6, cfg=3)
    nq = len(P["quad_conn"])
    q = np.full(nq, 2e3)
    w = np.full(nq, 2400.0 * W.GRAV)
    f = L.area_load(P, q, w, np.array([0.0, 0.0, -1.0]))
    assert np.allclose(f, P["f"], rtol=1e-12, atol=1e-12 * np.abs(P["f"]).max())


@pytest.mark.parametrize("make,s", [(lambda: W.tiny_shell(2, 0), 1.0), (lambda: W.tiny_shell(3, 5), 0.5)])
def test_gradient_vs_global_complex_step(make, s):
    P = make()
    q, w, d = _load_case(P, 1)
    u, f = L.evaluate(P, q, w, d)
    dX, dt = L.compliance_gradient(P, u, q, w, d, s)
    nn = len(P["x"])
    for (n, a) in [(nn // 2, 2), (1, 0), (nn - 2, 1), (nn // 2 + 1, 0)]:
        ref = L.global_complex_step(P, q, w, d, "xyz", (n, a), s)
        assert abs(dX[a, n] - ref) <= 1e-10 * max(abs(ref), 1e-6 * np.abs(dX).max())
    for e in (0, len(dt) - 1):
        ref = L.global_complex_step(P, q, w, d, "t", e, s)
        assert abs(dt[e] - ref) <= 1e-10 * max(abs(ref), 1e-6 * np.abs(dt).max())
    # the load term matters: the fixed-load gradient misses it
    dX0, _ = Gd.adjoint_gradient(P, u, s)
    assert np.abs(dX - dX0).max() > 1e-3 * np.abs(dX).max()
