"""Oracle: global assembly, CSR pattern, scatter map and supports (test infrastructure only).

PAPER.md:58 and :83 — every element's local matrix is added into the global K
(JAX-SSO vmaps the element functions and builds a BCOO matrix whose duplicate
entries are summed); PAPER.md:82 — `element_K_*_indices` give the global row
and column of each element entry.  SURVEY.md §8(c) C3 fixes the plain
definition used here (reading c8):

  * a Python dict keyed by (row, col); every (a, b) pair of every element is
    inserted, even when its value is 0.0 (structural pattern);
  * element DOF list [6 node + c]; values summed in ascending element order
    (beams first, then quads);
  * CSR = keys sorted by (row, col): row_ptr int64, col_idx int32;
  * scatter map pos[e][a][b] = index of (dof_a, dof_b) in the CSR by binary
    search; block rank[e][i][j] = position of node j in the sorted node
    adjacency of node i.

Supports (Eqs. 2-3; reading c1): the paper imposes
Vu = b with Lagrange multipliers.  With b = 0 the same u follows from
symmetric elimination, which keeps K SPD for CG:
constrained row/column set to 0 except the diagonal, kept (1.0 if it is 0).
`lagrange_system` builds the paper's augmented form for the equivalence pin.

Pins: tests/test_oracle_assembly.py — brute-force node-pair sets, the grid nnz
closed form, K·(rigid translation) = 0, element-order shuffle invariance,
Lagrange-vs-elimination equivalence (tests/test_oracle_solve.py).
"""
from __future__ import annotations

import bisect
import numpy as np

from . import beam as _beam
from . import shell as _shell


def n_beams(P):
    return len(P["beam_conn"])


def n_quads(P):
    return len(P["quad_conn"])


def element_nodes(P, e):
    """Element e in the global element order: beams first, then quads."""
    nb = n_beams(P)
    if e < nb:
        return [int(v) for v in P["beam_conn"][e]]
    return [int(v) for v in P["quad_conn"][e - nb]]


def element_dofs(nodes):
    """DOF list [6 node + c] (node-major, component-minor)."""
    return [6 * n + c for n in nodes for c in range(6)]


def node_xyz(P, n, override=None):
    if override is not None:
        return override[n]
    return np.array([P["x"][n], P["y"][n], P["z"][n]])


def coords(P):
    return np.stack([P["x"], P["y"], P["z"]], axis=1)


def shear_modulus(P, e):
    if P.get("G") is not None:
        return P["G"][e]
    return P["E"][e] / (2.0 * (1.0 + P["nu"][e]))


def element_K(P, e, X=None, t=None):
    """Global element matrix of element e.  X: optional [n_nodes, 3] coordinate
    array (may be complex), t: optional per-quad thickness array."""
    if X is None:
        X = coords(P)
    nb = n_beams(P)
    nodes = element_nodes(P, e)
    if e < nb:
        return _beam.beam_K(X[nodes[0]], X[nodes[1]], P["E"][e], shear_modulus(P, e),
                            P["A"][e], P["Iy"][e], P["Iz"][e], P["J"][e])
    q = e - nb
    tq = P["t"][q] if t is None else t[q]
    return _shell.shell_K(X[nodes], tq, P["E"][e], P["nu"][e])


def assemble_dok(P, X=None, t=None, order=None):
    """Dict-of-keys assembly; values summed in ascending element order (or in
    `order`, used only by the shuffle-invariance pin)."""
    ne = n_beams(P) + n_quads(P)
    dok = {}
    for e in (range(ne) if order is None else order):
        Ke = element_K(P, e, X, t)
        dofs = element_dofs(element_nodes(P, e))
        for a, ra in enumerate(dofs):
            for b, cb in enumerate(dofs):
                key = (ra, cb)
                dok[key] = dok.get(key, 0.0) + Ke[a, b]
    return dok


def csr_from_dok(dok, ndof):
    """CSR = keys sorted by (row, col); row_ptr int64, col_idx int32."""
    keys = sorted(dok.keys())
    vals = np.array([dok[k] for k in keys])
    rows = np.array([k[0] for k in keys], dtype=np.int64)
    col_idx = np.array([k[1] for k in keys], dtype=np.int32)
    row_ptr = np.zeros(ndof + 1, dtype=np.int64)
    for r in rows:
        row_ptr[r + 1] += 1
    row_ptr = np.cumsum(row_ptr).astype(np.int64)
    return row_ptr, col_idx, vals


def dense_from_dok(dok, ndof, dtype=np.float64):
    K = np.zeros((ndof, ndof), dtype=dtype)
    for (r, c), v in dok.items():
        K[r, c] = v
    return K


def scatter_map(P, row_ptr, col_idx):
    """pos[e][a][b] = CSR index of (dof_a, dof_b), by binary search in the row."""
    ne = n_beams(P) + n_quads(P)
    out = []
    cols = col_idx.tolist()
    for e in range(ne):
        dofs = element_dofs(element_nodes(P, e))
        m = len(dofs)
        pos = np.zeros((m, m), dtype=np.int64)
        for a, ra in enumerate(dofs):
            lo, hi = int(row_ptr[ra]), int(row_ptr[ra + 1])
            for b, cb in enumerate(dofs):
                k = bisect.bisect_left(cols, cb, lo, hi)
                assert k < hi and cols[k] == cb
                pos[a, b] = k
        out.append(pos)
    return out


def node_adjacency(P):
    """Sorted node adjacency (incl. self): m in adj(n) iff n, m share an element."""
    nn = len(P["x"])
    adj = [set([n]) for n in range(nn)]
    ne = n_beams(P) + n_quads(P)
    for e in range(ne):
        nodes = element_nodes(P, e)
        for a in nodes:
            for b in nodes:
                adj[a].add(b)
    return [sorted(s) for s in adj]


def block_rank(P):
    """rank[e][i*k+j] = position of node j (element-local) in adj(node i)."""
    adj = node_adjacency(P)
    ne = n_beams(P) + n_quads(P)
    out = []
    for e in range(ne):
        nodes = element_nodes(P, e)
        r = []
        for a in nodes:
            for b in nodes:
                r.append(adj[a].index(b))
        out.append(r)
    return out


def fixed_dofs(P):
    """Support masks OR-merged per node (reading c7); returns a bool [6 n] array."""
    fixed = np.zeros(6 * len(P["x"]), dtype=bool)
    for n, m in zip(P["sup_node"], P["sup_mask"]):
        for c in range(6):
            if (int(m) >> c) & 1:
                fixed[6 * int(n) + c] = True
    return fixed


def apply_supports_dense(K, f, fixed):
    """zero constrained rows/columns except the diagonal,
    kept (1.0 if it is 0); f[c] = 0."""
    K = K.copy()
    f = f.copy()
    for c in np.nonzero(fixed)[0]:
        d = K[c, c]
        K[c, :] = 0.0
        K[:, c] = 0.0
        K[c, c] = d if d != 0.0 else 1.0
        f[c] = 0.0
    return K, f


def apply_supports_csr(row_ptr, col_idx, vals, fixed):
    """Elimination on CSR values (same rule as apply_supports_dense)."""
    vals = vals.copy()
    ndof = len(row_ptr) - 1
    for r in range(ndof):
        for k in range(int(row_ptr[r]), int(row_ptr[r + 1])):
            c = int(col_idx[k])
            if fixed[r] or fixed[c]:
                if r == c:
                    if vals[k] == 0.0:
                        vals[k] = 1.0
                else:
                    vals[k] = 0.0
    return vals


def lagrange_system(K, f, fixed, b=None):
    """PAPER.md Eq. 2: K_aug = [[K, V^T], [V, 0]], f_aug = (f; b), V u = b (Eq. 3);
    one row of V per constrained DOF with a single unit entry."""
    ndof = K.shape[0]
    cons = np.nonzero(fixed)[0]
    nbc = len(cons)
    V = np.zeros((nbc, ndof))
    for k, c in enumerate(cons):
        V[k, c] = 1.0
    Kaug = np.zeros((ndof + nbc, ndof + nbc), dtype=K.dtype)
    Kaug[:ndof, :ndof] = K
    Kaug[:ndof, ndof:] = V.T
    Kaug[ndof:, :ndof] = V
    faug = np.zeros(ndof + nbc, dtype=np.result_type(f, np.float64))
    faug[:ndof] = f
    if b is not None:
        faug[ndof:] = b
    return Kaug, faug


def incident_elements(P, n):
    """Elements containing node n, ascending (beams first, then quads)."""
    nb = n_beams(P)
    out = []
    if nb:
        out += [int(e) for e in np.nonzero((P["beam_conn"] == n).any(axis=1))[0]]
    if n_quads(P):
        out += [nb + int(q) for q in np.nonzero((P["quad_conn"] == n).any(axis=1))[0]]
    return out


def node_rows(P, n, X=None):
    """The six global rows 6n..6n+5 of the summed K (before supports), as a dict
    column -> 6-vector, summed over the incident elements in ascending order —
    the DOK definition restricted to one node (for full-size sampled checks)."""
    rows = {}
    for e in incident_elements(P, n):
        nodes = element_nodes(P, e)
        Ke = element_K(P, e, X)
        dofs = element_dofs(nodes)
        for il, nd in enumerate(nodes):
            if nd != n:
                continue
            for b, cb in enumerate(dofs):
                col = rows.setdefault(cb, np.zeros(6))
                col += Ke[6 * il:6 * il + 6, b]
    return rows
