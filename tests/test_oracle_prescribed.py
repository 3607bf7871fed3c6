"""Pins for oracle/prescribed.py (prescribed support displacements V u = b,
PAPER.md Eqs. 2-3; reading c18)."""
import numpy as np
import pytest

import workloads as W
from oracle import assembly as A, grad as Gd, prescribed as PR


def _b(P, seed):
    rng = np.random.default_rng(seed)
    b = np.zeros(6 * len(P["x"]))
    fixed = A.fixed_dofs(P)
    b[fixed] = rng.uniform(-1e-3, 1e-3, int(fixed.sum()))
    return b


@pytest.mark.parametrize("make,s", [(lambda: W.tiny_shell(2, 0), 1.0), (lambda: W.tiny_shell(3, 2), 0.5),
                                    (lambda: W.tiny_beam_grid(1), 1.0)])
def test_gradient_vs_complex_step_of_augmented_solve(make, s):
    P = make()
    b = _b(P, 3)
    u = PR.solve(P, b)
    fixed = A.fixed_dofs(P)
    assert np.allclose(u[fixed], b[fixed], rtol=0, atol=1e-15)
    dX, dt, _ = PR.gradient(P, u, s)
    nn = len(P["x"])
    for (n, a) in [(nn // 2, 2), (1, 0), (nn - 2, 1)]:
        ref = PR.global_complex_step(P, b, "xyz", (n, a), s)
        assert abs(dX[a, n] - ref) <= 1e-9 * max(abs(ref), 1e-6 * np.abs(dX).max())
    if len(dt):
        ref = PR.global_complex_step(P, b, "t", 1, s)
        assert abs(dt[1] - ref) <= 1e-9 * max(abs(ref), 1e-6 * np.abs(dt).max())


def test_zero_b_reduces_to_self_adjoint_gradient():
    P = W.tiny_shell(3, 1)
    u = PR.solve(P, np.zeros(6 * len(P["x"])))
    uc, _, _ = Gd.evaluate(P)
    assert np.allclose(u, uc, rtol=1e-10, atol=1e-12 * np.abs(uc).max())
    dX, dt, _ = PR.gradient(P, u, 1.0)
    gX, gt = Gd.adjoint_gradient(P, u, 1.0)
    assert np.allclose(dX, gX, rtol=1e-9, atol=1e-9 * np.abs(gX).max())


def test_rigid_translation_prescribed_everywhere_is_exact():
    # every node of a free plate constrained in translation to the same b: rotations free,
    # the plate translates rigidly, so u_trans = b, rotations = 0 and K u = 0.
    P = W.tiny_shell(2, 0, zamp=0.0)
    nn = len(P["x"])
    P = dict(P, sup_node=np.arange(nn, dtype=np.int32), sup_mask=np.full(nn, W.PINNED, np.uint8),
             f=np.zeros(6 * nn))
    b = np.zeros(6 * nn)
    for n in range(nn):
        b[6 * n:6 * n + 3] = [1e-3, -2e-3, 5e-4]
    u = PR.solve(P, b)
    ref = b.copy()
    assert np.allclose(u, ref, rtol=0, atol=1e-14)


def test_gradient_with_area_loads_vs_complex_step():
    from oracle import loads as L
    P = W.tiny_shell(3, 4)
    rng = np.random.default_rng(5)
    nq = len(P["quad_conn"])
    load = (rng.uniform(1e3, 3e3, nq), rng.uniform(2e4, 3e4, nq), np.array([0.1, 0.3, -1.0]))
    b = _b(P, 7)
    s = 0.5
    f = P["f"] + L.area_load(P, *load)
    u = PR.solve(P, b, f)
    dX, dt, _ = PR.gradient_with_loads(P, u, *load, s)
    nn = len(P["x"])
    for (n, a) in [(nn // 2, 2), (2, 0), (nn - 3, 1)]:
        ref = PR.global_complex_step(P, b, "xyz", (n, a), s, load)
        assert abs(dX[a, n] - ref) <= 1e-9 * max(abs(ref), 1e-6 * np.abs(dX).max())
    ref = PR.global_complex_step(P, b, "t", 2, s, load)
    assert abs(dt[2] - ref) <= 1e-9 * max(abs(ref), 1e-6 * np.abs(dt).max())
