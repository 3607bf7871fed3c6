"""Oracle: standard hat (linear cone) filter of sensitivities (test infrastructure only).

PAPER.md:280, 290, 349, 359: "we apply a standard hat filter with a radius of r to
the sensitivity" (citing Bletzinger 2014 for sensitivity filtering).  The paper
gives no formula; reading (DESIGN.md c16): the normalised linear-hat convolution
over the points within distance r,

    out_i = sum_j w_ij in_j / sum_j w_ij,   w_ij = max(0, r - |X_i - X_j|),

with X the node coordinates (node sensitivities) or the element centroids
(element sensitivities: mean of the element's node coordinates).  Brute force
over all pairs, ascending j.

Pins (tests/test_oracle_filter.py): constants are preserved; r below the point
spacing is the identity; the weighted sum sum_i W_i out_i = sum_i W_i in_i
(W_i = sum_j w_ij) holds because w is symmetric; a linear field is reproduced at
points whose neighbourhood is symmetric.
"""
from __future__ import annotations

import numpy as np


def points(P, on_elements):
    X = np.stack([P["x"], P["y"], P["z"]], axis=1)
    if not on_elements:
        return X
    conns = [c for c in (P["beam_conn"], P["quad_conn"]) if len(c)]
    cents = []
    for c in conns:
        for el in c:
            cents.append(X[list(el)].mean(axis=0))
    return np.array(cents)


def hat_filter_rows(P, radius, values, rows, on_elements=False):
    """The same definition for selected output points only (sampled checks at sizes
    where the all-pairs loop is too slow); the sum over j is vectorised.
    values [ncomp, n] (or [n]) -> [ncomp, len(rows)] (or [len(rows)])."""
    X = points(P, on_elements)
    v = np.atleast_2d(np.asarray(values, dtype=np.float64))
    out = np.zeros((v.shape[0], len(rows)))
    for k, i in enumerate(rows):
        d = np.sqrt(np.sum((X - X[i]) ** 2, axis=1))
        w = np.maximum(0.0, radius - d)
        out[:, k] = (v * w).sum(axis=1) / w.sum()
    return out if np.ndim(values) > 1 else out[0]


def hat_filter(P, radius, values, on_elements=False):
    """values [ncomp, n] (or [n]) -> filtered, same shape."""
    X = points(P, on_elements)
    v = np.atleast_2d(np.asarray(values, dtype=np.float64))
    n = len(X)
    out = np.zeros_like(v)
    for i in range(n):
        num = np.zeros(v.shape[0])
        den = 0.0
        for j in range(n):
            d = np.sqrt(np.sum((X[i] - X[j]) ** 2))
            w = radius - d
            if w > 0.0:
                num += w * v[:, j]
                den += w
        out[:, i] = num / den
    return out.reshape(np.shape(values))
