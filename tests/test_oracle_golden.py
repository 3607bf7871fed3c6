"""Golden values: the paper's printed numbers and closed-form worked values.

tests/golden/closed_form.txt pins the oracle (asserted).
tests/golden/paper_validation.txt holds PAPER.md's barrel-arch numbers.  Under
the readings of DESIGN.md (c4 element details, c14 "500 N" load) the oracle
does NOT reproduce them (SE 188 vs 1229.7 N m): the paper's geometry, mesh
and element details are not recoverable from the text.  That comparison is
kept as a strict xfail so the discrepancy stays visible; the element itself
is pinned by the closed-form and invariant tests instead ("parity unpinned"
against the paper's absolute barrel values).
"""
import math
import os

import numpy as np
import pytest

import workloads as W
from oracle import grad as Gd

HERE = os.path.join(os.path.dirname(__file__), "golden")


def load(name):
    out = {}
    with open(os.path.join(HERE, name)) as fh:
        for line in fh:
            line = line.split("#")[0].strip()
            if line:
                k, v = line.split("=")
                out[k.strip()] = float(v)
    return out


def test_closed_form_cantilever_values():
    g = load("closed_form.txt")
    E, I, A, J, L, Pld = 210e9, 1e-6, 1e-3, 2e-6, 2.5, 1000.0
    Gm = E / 2.6
    x = np.array([0.0, L])
    f = np.zeros(12)
    f[8] = Pld          # tip load along global Z
    f[6] = Pld          # axial tip load
    f[9] = Pld          # torsion about the axis
    P = W._problem("cant", x, np.zeros(2), np.zeros(2), beam_conn=np.array([[0, 1]]),
                   A=[A], Iy=[I], Iz=[I], J=[J], E=[E], nu=[0.3], G=[Gm],
                   sup_node=[0], sup_mask=[W.CLAMPED], f=f)
    u, _, _ = Gd.evaluate(P)
    assert u[8] == pytest.approx(g["cantilever_tip_w_m"], rel=1e-5)
    assert abs(u[10]) == pytest.approx(g["cantilever_tip_rot"], rel=1e-5)
    assert u[6] == pytest.approx(g["cantilever_axial_m"], rel=1e-5)
    assert u[9] == pytest.approx(g["cantilever_torsion_rad"], rel=1e-5)
    assert Pld * u[8] == pytest.approx(g["cantilever_compliance_Nm"], rel=1e-5)


def test_navier_coefficient_value():
    g = load("closed_form.txt")
    s = 0.0
    for m in range(1, 400, 2):
        for n in range(1, 400, 2):
            s += (-1) ** ((m - 1) // 2 + (n - 1) // 2) / (m * n * (m * m + n * n) ** 2)
    assert 16 / math.pi ** 6 * s == pytest.approx(g["navier_kirchhoff_coeff"], rel=1e-4)


@pytest.mark.xfail(strict=True, reason="paper barrel-arch geometry/element not recoverable "
                                       "(DESIGN.md reading c14); parity unpinned vs paper")
def test_paper_barrel_arch_strain_energy():
    g = load("paper_validation.txt")
    P = W.barrel_arch(500.0)
    u, _, _ = Gd.evaluate(P)
    se = 0.5 * float(P["f"] @ u)
    assert se == pytest.approx(g["barrel_strain_energy_Nm"], rel=0.03)
