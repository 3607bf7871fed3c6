"""Pins for oracle/beam.py against closed-form Euler-Bernoulli mechanics.

Euler-Bernoulli frame elements are nodally exact for end loads, so a
cantilever of any number of elements reproduces the textbook tip results
(SPEC.md:150-152, 293):
    tip deflection PL^3 / (3 E I), tip rotation PL^2 / (2 E I),
    axial PL / (E A), torsion T L / (G J).
"""
import math

import numpy as np
import pytest

import workloads as W
from oracle import assembly as A, beam, grad as Gd

E, NU = 210e9, 0.3
G = E / (2 * (1 + NU))
SEC = dict(A=1e-3, Iy=2e-6, Iz=1e-6, J=2e-6)


def cantilever(direction, m, L, tip_load6, Iy=SEC["Iy"], Iz=SEC["Iz"]):
    d = np.asarray(direction, float)
    d = d / np.linalg.norm(d)
    pts = np.array([k * L / m * d for k in range(m + 1)]) + np.array([0.3, -0.2, 0.1])
    conn = [(k, k + 1) for k in range(m)]
    f = np.zeros(6 * (m + 1))
    f[6 * m:6 * m + 6] = tip_load6
    return W._problem("cant", pts[:, 0], pts[:, 1], pts[:, 2], beam_conn=np.array(conn),
                      A=np.full(m, SEC["A"]), Iy=np.full(m, Iy), Iz=np.full(m, Iz),
                      J=np.full(m, SEC["J"]), E=np.full(m, E), nu=np.full(m, NU), G=None,
                      sup_node=[0], sup_mask=[W.CLAMPED], f=f)


def perp(d):
    d = np.asarray(d, float) / np.linalg.norm(d)
    a = np.array([0.3, 0.5, 0.7])
    v = a - a.dot(d) * d
    return v / np.linalg.norm(v)


@pytest.mark.parametrize("m", [1, 3])
@pytest.mark.parametrize("direction", [(1, 0, 0), (0.3, -0.8, 0.5), (0.1, 0.2, -1.0)])
def test_cantilever_transverse_isotropic(m, direction):
    # Iy = Iz: any transverse tip load gives PL^3/(3EI) along the load, whatever the roll
    L, Pld, I = 2.5, 1000.0, 1e-6
    n = perp(direction)
    load = np.zeros(6)
    load[:3] = Pld * n
    P = cantilever(direction, m, L, load, Iy=I, Iz=I)
    u, _, _ = Gd.evaluate(P)
    tip = u[6 * m:6 * m + 3]
    w = tip.dot(n)
    assert w == pytest.approx(Pld * L ** 3 / (3 * E * I), rel=1e-10)
    # no component along the axis or the third direction
    d = np.asarray(direction, float) / np.linalg.norm(direction)
    assert abs(tip.dot(d)) < 1e-10 * abs(w)
    # tip rotation magnitude PL^2/(2EI), about d x n
    rot = u[6 * m + 3:6 * m + 6]
    assert np.linalg.norm(rot) == pytest.approx(Pld * L ** 2 / (2 * E * I), rel=1e-10)
    assert rot.dot(np.cross(d, n)) > 0  # right-hand rule: load along n rotates about d x n


@pytest.mark.parametrize("m", [1, 4])
def test_cantilever_axial_and_torsion(m):
    L, Pld, T = 2.5, 1000.0, 1000.0
    d = np.array([0.2, 0.9, -0.4])
    d /= np.linalg.norm(d)
    load = np.zeros(6)
    load[:3] = Pld * d
    load[3:] = T * d
    P = cantilever(d, m, L, load)
    u, _, _ = Gd.evaluate(P)
    assert u[6 * m:6 * m + 3].dot(d) == pytest.approx(Pld * L / (E * SEC["A"]), rel=1e-10)
    assert u[6 * m + 3:6 * m + 6].dot(d) == pytest.approx(T * L / (G * SEC["J"]), rel=1e-10)


def test_cantilever_roll_convention_Iy_Iz():
    # reading c6 / C1: member along global X -> local z = global Z (aux = Z), so a Z tip
    # load bends about local y (uses Iy) and a Y tip load bends about local z (uses Iz).
    L, Pld = 2.0, 500.0
    for comp, I in ((2, SEC["Iy"]), (1, SEC["Iz"])):
        load = np.zeros(6)
        load[comp] = Pld
        P = cantilever((1, 0, 0), 2, L, load)
        u, _, _ = Gd.evaluate(P)
        assert u[6 * 2 + comp] == pytest.approx(Pld * L ** 3 / (3 * E * I), rel=1e-10)
    # vertical member: aux falls back to global X (|e_x . Z| > cos 1e-6)
    R, _ = beam.beam_frame(np.zeros(3), np.array([0.0, 0.0, 3.0]))
    assert np.allclose(R[2], [1.0, 0.0, 0.0])


def test_closed_form_worked_values():
    # SURVEY.md §8(d) "closed-form worked values": C1 section, L = 2.5, P = 1 kN
    L, Pld, I = 2.5, 1000.0, 1e-6
    load = np.zeros(6)
    load[2] = Pld
    P = cantilever((1, 0, 0), 1, L, load, Iy=I, Iz=I)
    u, _, _ = Gd.evaluate(P)
    assert u[8] == pytest.approx(2.48016e-2, rel=1e-5)
    assert Gd.compliance(P["f"], u) == pytest.approx(24.8016, rel=1e-5)


def rigid_modes_global(X):
    c = X.mean(axis=0)
    modes = []
    for k in range(3):
        r = np.zeros(6 * len(X))
        r[k::6] = 1.0
        modes.append(r)
    for k in range(3):
        w = np.zeros(3)
        w[k] = 1.0
        r = np.zeros(6 * len(X))
        for i, Xi in enumerate(X):
            r[6 * i:6 * i + 3] = np.cross(w, Xi - c)
            r[6 * i + 3:6 * i + 6] = w
        modes.append(r)
    return modes


def test_beam_rigid_modes_and_symmetry():
    rng = np.random.default_rng(7)
    for _ in range(5):
        Xi, Xj = rng.normal(size=3), rng.normal(size=3)
        K = beam.beam_K(Xi, Xj, E, G, 1e-3, 2e-6, 1e-6, 3e-6)
        assert np.abs(K - K.T).max() <= 1e-14 * np.abs(K).max()
        for r in rigid_modes_global(np.array([Xi, Xj])):
            assert np.linalg.norm(K @ r) <= 1e-12 * np.linalg.norm(K) * np.linalg.norm(r)
        ev = np.linalg.eigvalsh(K)
        assert ev[0] > -1e-9 * ev[-1]
        K2 = beam.beam_K(Xi, Xj, 2 * E, 2 * G, 1e-3, 2e-6, 1e-6, 3e-6)
        assert np.array_equal(K2, 2 * K)
