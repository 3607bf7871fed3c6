"""Pins for oracle/filter.py (hat filter of sensitivities)."""
import numpy as np
import pytest

import workloads as W
from oracle import filter as F


@pytest.mark.parametrize("on_elements", [False, True])
def test_hat_filter_properties(on_elements):
    P = W.tiny_shell(5, seed=2, L=5.0, zamp=0.2)
    X = F.points(P, on_elements)
    n = len(X)
    rng = np.random.default_rng(0)
    # constants preserved
    assert np.allclose(F.hat_filter(P, 2.2, np.full(n, 3.5), on_elements), 3.5, rtol=1e-14)
    # radius below the spacing: identity
    v = rng.standard_normal(n)
    assert np.array_equal(F.hat_filter(P, 0.5, v, on_elements), v)
    # symmetric weights: sum_i W_i out_i == sum_i W_i in_i
    r = 2.2
    out = F.hat_filter(P, r, v, on_elements)
    Wt = np.array([np.sum(np.maximum(0.0, r - np.linalg.norm(X - X[i], axis=1))) for i in range(n)])
    assert np.dot(Wt, out) == pytest.approx(np.dot(Wt, v), rel=1e-12)
    # multi-component input filters each component
    v3 = rng.standard_normal((3, n))
    o3 = F.hat_filter(P, r, v3, on_elements)
    assert np.allclose(o3[1], F.hat_filter(P, r, v3[1], on_elements), rtol=1e-15)


def test_hat_filter_reproduces_linear_field_on_symmetric_patch():
    # flat regular grid: an interior node with a complete neighbourhood keeps a linear field
    P = W.tiny_shell(8, seed=0, L=8.0, zamp=0.0)
    X = F.points(P, False)
    v = 2.0 * X[:, 0] - 0.5 * X[:, 1] + 1.0
    out = F.hat_filter(P, 1.5, v)
    centre = 4 * 9 + 4
    assert out[centre] == pytest.approx(v[centre], rel=1e-13)


def test_sampled_rows_match_full_filter():
    P = W.tiny_shell(4, seed=3, L=4.0, zamp=0.3)
    v = np.random.default_rng(2).standard_normal((2, len(P["quad_conn"])))
    full = F.hat_filter(P, 1.7, v, True)
    rows = [0, 5, 15]
    assert np.allclose(F.hat_filter_rows(P, 1.7, v, rows, True), full[:, rows], rtol=1e-13, atol=0)
