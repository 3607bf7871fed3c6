"""Oracle: 3D Euler-Bernoulli frame element, 12x12 (test infrastructure only).

Follows PAPER.md:75 (`element_K_bc_local`) and PAPER.md:112 (a beam-column
is defined by E, G, Iy, Iz, J, A and two nodes), with the local-axis,
DOF-order and sign conventions of SURVEY.md §8(c) C1 (reading c6).
All functions accept complex inputs so that derivatives can be taken by
complex step (no abs(), no np.linalg.norm on complex values; branches on real
parts only).

Pins: tests/test_oracle_beam.py — cantilever tip deflection PL^3/(3EI),
tip rotation PL^2/(2EI), axial PL/(EA), torsion TL/(GJ) for arbitrary member
orientation; six exact rigid-body modes; symmetry.
"""
from __future__ import annotations

import math
import numpy as np


def _dot(a, b):
    return a[0] * b[0] + a[1] * b[1] + a[2] * b[2]


def _cross(a, b):
    return np.array([a[1] * b[2] - a[2] * b[1],
                     a[2] * b[0] - a[0] * b[2],
                     a[0] * b[1] - a[1] * b[0]], dtype=np.result_type(a, b))


def _sqrt(v):
    # analytic square root (works for complex-step perturbed values)
    return np.sqrt(v)


def beam_frame(Xi, Xj):
    """Local axes (reading C1): e_x along the member; auxiliary a = global Z
    unless |e_x . Z| > cos(1e-6) (then global X); e_z = normalise(a - (a.e_x)e_x);
    e_y = e_z x e_x.  Returns (R, L) with rows of R = (e_x, e_y, e_z)."""
    d = Xj - Xi
    L = _sqrt(_dot(d, d))
    ex = d / L
    a = np.array([0.0, 0.0, 1.0])
    if abs(np.real(ex[2])) > math.cos(1e-6):
        a = np.array([1.0, 0.0, 0.0])
    w = a - _dot(a, ex) * ex
    ez = w / _sqrt(_dot(w, w))
    ey = _cross(ez, ex)
    R = np.array([ex, ey, ez])
    return R, L


def beam_k_local(E, G, A, Iy, Iz, J, L):
    """12x12 local stiffness, local DOF order (u, v, w, th_x, th_y, th_z) per node
    (the standard frame matrix with right-hand rotation signs)."""
    dt = np.result_type(E, G, A, Iy, Iz, J, L, np.float64)
    k = np.zeros((12, 12), dtype=dt)
    # axial
    k[0, 0] = k[6, 6] = E * A / L
    k[0, 6] = -E * A / L
    # torsion
    k[3, 3] = k[9, 9] = G * J / L
    k[3, 9] = -G * J / L
    # bending in local x-y plane: v (1, 7), th_z (5, 11), uses Iz
    k[1, 1] = k[7, 7] = 12.0 * E * Iz / L ** 3
    k[1, 7] = -12.0 * E * Iz / L ** 3
    k[1, 5] = k[1, 11] = 6.0 * E * Iz / L ** 2
    k[5, 7] = k[7, 11] = -6.0 * E * Iz / L ** 2
    k[5, 5] = k[11, 11] = 4.0 * E * Iz / L
    k[5, 11] = 2.0 * E * Iz / L
    # bending in local x-z plane: w (2, 8), th_y (4, 10), uses Iy
    k[2, 2] = k[8, 8] = 12.0 * E * Iy / L ** 3
    k[2, 8] = -12.0 * E * Iy / L ** 3
    k[2, 4] = k[2, 10] = -6.0 * E * Iy / L ** 2
    k[4, 8] = k[8, 10] = 6.0 * E * Iy / L ** 2
    k[4, 4] = k[10, 10] = 4.0 * E * Iy / L
    k[4, 10] = 2.0 * E * Iy / L
    # symmetry: copy the upper triangle to the lower one
    for a in range(12):
        for b in range(a + 1, 12):
            k[b, a] = k[a, b]
    return k


def beam_K(Xi, Xj, E, G, A, Iy, Iz, J):
    """Global 12x12 stiffness K_e = T^T k_loc T, T = blockdiag(R, R, R, R)."""
    R, L = beam_frame(np.asarray(Xi), np.asarray(Xj))
    k = beam_k_local(E, G, A, Iy, Iz, J, L)
    dt = np.result_type(k, R)
    T = np.zeros((12, 12), dtype=dt)
    for b in range(4):
        T[3 * b:3 * b + 3, 3 * b:3 * b + 3] = R
    return T.T @ k @ T
