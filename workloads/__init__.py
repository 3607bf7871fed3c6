"""Seeded synthetic inputs shared by the oracle and the CUDA path.

This module holds INPUT GENERATION ONLY: node coordinates, connectivity,
sections, materials, supports and lumped nodal loads.  It contains none of
the method's arithmetic (no element stiffness, assembly, solve or gradient),
so the oracle (`oracle/`) and the product path (`paper_2407_20026_b200/`) can
both consume it without sharing any code of the method.

Recipes follow SURVEY.md §8(d) (generator table) and the readings listed in
DESIGN.md ("Input recipe").  The paper's own workloads (PAPER.md:144-145,
197, 272-291) have no public data; these stand in for them with the shapes
and distributions of BASELINE.json `configs`.

Every generator returns a `Problem` dict with fp64 / int32 / uint8 numpy
arrays:

    x, y, z        float64 [n_nodes]           node coordinates (SoA)
    beam_conn      int32   [n_beams, 2]
    quad_conn      int32   [n_quads, 4]        cyclic order, CCW from +z
    A, Iy, Iz, J   float64 [n_beams]           beam sections
    t              float64 [n_quads]           shell thickness
    E, nu          float64 [n_beams + n_quads] beams first, then quads
    G              float64 [n_beams + n_quads] or None (-> E / (2 (1 + nu)))
    sup_node       int32   [n_sup]             supported node ids
    sup_mask       uint8   [n_sup]             bit c set = DOF c fixed (b = 0)
    f              float64 [6 n_nodes]         nodal load vector
    name           str

DOF numbering is node-major, component-minor: 6*i + c with
c in (UX, UY, UZ, RX, RY, RZ).
"""
from __future__ import annotations

import math
import numpy as np

SEED_ROOT = 240720026          # SeedSequence([240720026, cfg, design])
GRAV = 9.81                    # m/s^2, SURVEY.md §8(c) c11

PINNED = 0b000111              # UX, UY, UZ fixed (reading c9)
CLAMPED = 0b111111             # all 6 DOF fixed (reading c9)


def _rng(cfg: int, design: int = 0) -> np.random.Generator:
    return np.random.default_rng(np.random.SeedSequence([SEED_ROOT, cfg, design]))


# ----------------------------------------------------------------------------
# mesh helpers (connectivity only)
# ----------------------------------------------------------------------------

def grid_nodes(n: int, L: float = 10.0, origin=(0.0, 0.0)):
    """Node (i, j) -> index j*(n+1)+i at (origin + i L/n, origin + j L/n)."""
    i = np.tile(np.arange(n + 1), n + 1)
    j = np.repeat(np.arange(n + 1), n + 1)
    x = origin[0] + i * (L / n)
    y = origin[1] + j * (L / n)
    return x.astype(np.float64), y.astype(np.float64)


def grid_quads(n: int) -> np.ndarray:
    """Element (i, j) -> index j*n+i with nodes [a, a+1, a+n+2, a+n+1], a = j(n+1)+i."""
    i = np.tile(np.arange(n), n)
    j = np.repeat(np.arange(n), n)
    a = j * (n + 1) + i
    return np.stack([a, a + 1, a + n + 2, a + n + 1], axis=1).astype(np.int32)


def boundary_nodes(n: int) -> np.ndarray:
    ids = []
    for j in range(n + 1):
        for i in range(n + 1):
            if i == 0 or j == 0 or i == n or j == n:
                ids.append(j * (n + 1) + i)
    return np.asarray(ids, dtype=np.int32)


def lumped_vertical_load(x, y, z, quad_conn, q, rho_g_t=None):
    """Reading c11: vertical -Z loads, A_e = 1/2 |(X3-X1) x (X4-X2)|, each node
    gets q A_e / 4 (pressure) + rho g t_e A_e / 4 (self-weight).  This is a
    load model (an input), not part of the method's arithmetic."""
    X = np.stack([x, y, z], axis=1)
    c = quad_conn
    d1 = X[c[:, 2]] - X[c[:, 0]]
    d2 = X[c[:, 3]] - X[c[:, 1]]
    Ae = 0.5 * np.linalg.norm(np.cross(d1, d2), axis=1)
    w = q * Ae / 4.0
    if rho_g_t is not None:
        w = w + rho_g_t * Ae / 4.0
    fz = np.zeros(x.shape[0])
    for k in range(4):
        np.add.at(fz, c[:, k], -w)
    f = np.zeros(6 * x.shape[0])
    f[2::6] = fz
    return f


def _fourier_field(x, y, L, rng, n_modes):
    """Sum of n_modes random sin-sin modes; (m_k, n_k) ~ U{1..4}^2, c_k ~ U(-1, 1)."""
    m = rng.integers(1, 5, size=n_modes)
    nn = rng.integers(1, 5, size=n_modes)
    c = rng.uniform(-1.0, 1.0, size=n_modes)
    out = np.zeros_like(x)
    for k in range(n_modes):
        out += c[k] * np.sin(m[k] * math.pi * x / L) * np.sin(nn[k] * math.pi * y / L)
    return out


def _problem(name, x, y, z, *, beam_conn=None, quad_conn=None, A=None, Iy=None, Iz=None,
             J=None, t=None, E=None, nu=None, G=None, sup_node, sup_mask, f):
    nb = 0 if beam_conn is None else len(beam_conn)
    nq = 0 if quad_conn is None else len(quad_conn)
    P = dict(
        name=name,
        x=np.ascontiguousarray(x, np.float64), y=np.ascontiguousarray(y, np.float64),
        z=np.ascontiguousarray(z, np.float64),
        beam_conn=np.zeros((0, 2), np.int32) if beam_conn is None else np.ascontiguousarray(beam_conn, np.int32),
        quad_conn=np.zeros((0, 4), np.int32) if quad_conn is None else np.ascontiguousarray(quad_conn, np.int32),
        A=np.zeros(0) if A is None else np.ascontiguousarray(A, np.float64),
        Iy=np.zeros(0) if Iy is None else np.ascontiguousarray(Iy, np.float64),
        Iz=np.zeros(0) if Iz is None else np.ascontiguousarray(Iz, np.float64),
        J=np.zeros(0) if J is None else np.ascontiguousarray(J, np.float64),
        t=np.zeros(0) if t is None else np.ascontiguousarray(t, np.float64),
        E=np.ascontiguousarray(E, np.float64), nu=np.ascontiguousarray(nu, np.float64),
        G=None if G is None else np.ascontiguousarray(G, np.float64),
        sup_node=np.ascontiguousarray(sup_node, np.int32),
        sup_mask=np.ascontiguousarray(sup_mask, np.uint8),
        f=np.ascontiguousarray(f, np.float64),
    )
    assert P["E"].shape == (nb + nq,) and P["nu"].shape == (nb + nq,)
    return P


# ----------------------------------------------------------------------------
# BASELINE.json configs
# ----------------------------------------------------------------------------

def config1():
    """C1 grid-shell (beams only), BASELINE.json configs[0]; SURVEY.md §8(d) C1."""
    rng = _rng(1)
    xs = -5.0 + 2.5 * np.arange(5)
    x = np.tile(xs, 5)
    y = np.repeat(xs, 5)
    z = 2.0 * (1.0 - (x * x + y * y) / 50.0)
    corners = [0, 4, 20, 24]
    for k in range(25):
        if k not in corners:
            z[k] += rng.uniform(-0.05, 0.05)
    conn = []
    for j in range(5):
        for i in range(4):
            conn.append((j * 5 + i, j * 5 + i + 1))
    for j in range(4):
        for i in range(5):
            conn.append((j * 5 + i, (j + 1) * 5 + i))
    nb = len(conn)
    E = np.full(nb, 210e9)
    nu = np.full(nb, 0.3)
    G = E / 2.6
    f = np.zeros(6 * 25)
    for k in range(25):
        if k not in corners:
            f[6 * k + 2] = -1000.0
    return _problem("C1", x, y, z, beam_conn=np.array(conn), A=np.full(nb, 1e-3),
                    Iy=np.full(nb, 1e-6), Iz=np.full(nb, 1e-6), J=np.full(nb, 2e-6),
                    E=E, nu=nu, G=G, sup_node=corners, sup_mask=[PINNED] * 4, f=f)


def config2():
    """C2 shallow shell 20x20, BASELINE.json configs[1]; SURVEY.md §8(d) C2."""
    n, L = 20, 10.0
    rng = _rng(2)
    x, y = grid_nodes(n, L)
    z = 1.5 * np.sin(math.pi * x / L) * np.sin(math.pi * y / L)
    conn = grid_quads(n)
    nq = len(conn)
    t = 0.1 * (1.0 + rng.uniform(-0.1, 0.1, size=nq))
    bnd = boundary_nodes(n)
    f = lumped_vertical_load(x, y, z, conn, 5e3)
    return _problem("C2", x, y, z, quad_conn=conn, t=t, E=np.full(nq, 30e9), nu=np.full(nq, 0.2),
                    sup_node=bnd, sup_mask=np.full(len(bnd), PINNED), f=f)


def shell_config3(n: int, cfg: int = 3, supports: str = "clamped_edges", L: float = 10.0, design: int = 0):
    """C3 / C3b / C4 shell family, SURVEY.md §8(d) C3, C3b, C4.

    z = 1.5 sin sin + dz, dz = s * sum of 8 Fourier modes scaled to max|dz| = 0.2 m;
    t ~ log-uniform [0.05, 0.2]; E = 30 GPa, nu = 0.2; self-weight rho = 2400 kg/m^3
    plus 2 kN/m^2.  supports: 'clamped_edges' (C3) or 'c4' (edge y=0 clamped, corners
    (0, L), (L, L) pinned).  design > 0 draws another seeded instance of the recipe
    (design 0 is the configuration itself)."""
    rng = _rng(cfg, design)
    x, y = grid_nodes(n, L)
    dz = _fourier_field(x, y, L, rng, 8)
    amax = np.max(np.abs(dz))
    dz = dz * (0.2 / amax) if amax > 0 else dz
    z = 1.5 * np.sin(math.pi * x / L) * np.sin(math.pi * y / L) + dz
    conn = grid_quads(n)
    nq = len(conn)
    t = np.exp(rng.uniform(math.log(0.05), math.log(0.2), size=nq))
    f = lumped_vertical_load(x, y, z, conn, 2e3, rho_g_t=2400.0 * GRAV * t)
    if supports == "clamped_edges":
        sn = boundary_nodes(n)
        sm = np.full(len(sn), CLAMPED)
    elif supports == "c4":
        sn = list(range(n + 1)) + [n * (n + 1), n * (n + 1) + n]
        sm = [CLAMPED] * (n + 1) + [PINNED, PINNED]
    else:
        raise ValueError(supports)
    return _problem(f"C{cfg}-n{n}", x, y, z, quad_conn=conn, t=t, E=np.full(nq, 30e9),
                    nu=np.full(nq, 0.2), sup_node=sn, sup_mask=sm, f=f)


def config3():
    return shell_config3(200, cfg=3)


def config3b():
    """The '1M DOF' metric point (reading c15): C3 recipe at n = 408 -> 1 003 686 DOF."""
    return shell_config3(408, cfg=3)


def config4():
    return shell_config3(1000, cfg=4, supports="c4")


def config5_design(b: int, n: int = 50, L: float = 10.0):
    """C5 design b: z_b = sum of 6 Fourier modes scaled to max|z| = a_b ~ U(0.5, 1.0);
    t ~ U(0.05, 0.3) i.i.d.; corners pinned; q = 5 kN/m^2."""
    rng = _rng(5, b)
    x, y = grid_nodes(n, L)
    zf = _fourier_field(x, y, L, rng, 6)
    a_b = rng.uniform(0.5, 1.0)
    amax = np.max(np.abs(zf))
    z = zf * (a_b / amax)
    conn = grid_quads(n)
    nq = len(conn)
    t = rng.uniform(0.05, 0.3, size=nq)
    corners = [0, n, n * (n + 1), n * (n + 1) + n]
    f = lumped_vertical_load(x, y, z, conn, 5e3)
    return _problem(f"C5-d{b}", x, y, z, quad_conn=conn, t=t, E=np.full(nq, 30e9),
                    nu=np.full(nq, 0.2), sup_node=corners, sup_mask=[PINNED] * 4, f=f)


# ----------------------------------------------------------------------------
# paper validation geometry and tiny test meshes
# ----------------------------------------------------------------------------

def barrel_arch(load_per_node: float = 500.0):
    """PAPER.md:145 barrel arch: 19 m x 19 m plan, parabolic rise 4.5 m, 400 quads
    (20x20), E = 1.99e8 Pa, nu = 0.2, t = 0.25 m, ground lines pinned, downward
    nodal load at each node (reading c14: 500 N)."""
    n, L = 20, 19.0
    x, y = grid_nodes(n, L)
    z = 4.5 * (1.0 - ((x - 9.5) / 9.5) ** 2)
    conn = grid_quads(n)
    nq = len(conn)
    ground = [k for k in range((n + 1) ** 2) if (k % (n + 1)) in (0, n)]
    f = np.zeros(6 * (n + 1) ** 2)
    f[2::6] = -load_per_node
    return _problem("barrel", x, y, z, quad_conn=conn, t=np.full(nq, 0.25),
                    E=np.full(nq, 1.99e8), nu=np.full(nq, 0.2),
                    sup_node=ground, sup_mask=[PINNED] * len(ground), f=f)


def tiny_shell(n: int, seed: int = 0, L: float = 2.0, zamp: float = 0.3, supports="corners"):
    """Tiny seeded shell (SURVEY.md §8(d) closed-form list): random z in +-zamp,
    t in [0.05, 0.2], E = 30 GPa, nu = 0.2, corners pinned, random nodal loads."""
    rng = _rng(100 + n, seed)
    x, y = grid_nodes(n, L)
    z = rng.uniform(-zamp, zamp, size=x.shape[0])
    conn = grid_quads(n)
    nq = len(conn)
    t = rng.uniform(0.05, 0.2, size=nq)
    nn = (n + 1) ** 2
    f = rng.uniform(-1e3, 1e3, size=6 * nn)
    if supports == "corners":
        sn = [0, n, n * (n + 1), n * (n + 1) + n]
        sm = [PINNED] * 4
    elif supports == "edge":
        sn = list(range(n + 1))
        sm = [CLAMPED] * (n + 1)
    else:
        raise ValueError(supports)
    return _problem(f"tiny{n}-s{seed}", x, y, z, quad_conn=conn, t=t, E=np.full(nq, 30e9),
                    nu=np.full(nq, 0.2), sup_node=sn, sup_mask=sm, f=f)


def tiny_beam_grid(seed: int = 0):
    """3x3-node beam grid (12 beams) with seeded z, Iy = Iz."""
    rng = _rng(200, seed)
    xs = np.array([0.0, 1.0, 2.0])
    x = np.tile(xs, 3)
    y = np.repeat(xs, 3)
    z = rng.uniform(-0.3, 0.3, size=9)
    conn = []
    for j in range(3):
        for i in range(2):
            conn.append((j * 3 + i, j * 3 + i + 1))
    for j in range(2):
        for i in range(3):
            conn.append((j * 3 + i, (j + 1) * 3 + i))
    nb = len(conn)
    f = rng.uniform(-1e3, 1e3, size=6 * 9)
    return _problem(f"tinybeam-s{seed}", x, y, z, beam_conn=np.array(conn),
                    A=np.full(nb, 1e-3), Iy=np.full(nb, 1e-6), Iz=np.full(nb, 1e-6),
                    J=np.full(nb, 2e-6), E=np.full(nb, 210e9), nu=np.full(nb, 0.3), G=None,
                    sup_node=[0, 2, 6, 8], sup_mask=[PINNED] * 4, f=f)


def random_state(n_nodes: int, seed: int, scale: float = 1e-3) -> np.ndarray:
    """A seeded displacement-like vector u [6 n] used to test the gradient stage
    at full size with a state both sides take as input."""
    rng = _rng(300, seed)
    return rng.uniform(-scale, scale, size=6 * n_nodes)


CONFIGS = {
    "C1": config1,
    "C2": config2,
    "C3": config3,
    "C3b": config3b,
    "C4": config4,
}
