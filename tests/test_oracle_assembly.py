"""Pins for oracle/assembly.py (SURVEY.md §8(c) C3, C4, C10 'Assembly').

  * the CSR pattern equals the brute-force set of node pairs sharing an
    element (x 36 DOF pairs), on tiny beam, shell and mixed meshes;
  * nnz = 36 ((n+1)^2 + 4 n (n+1) + 4 n^2) on n x n quad grids;
  * the summed K annihilates global rigid translations AND rotations before
    supports (a transposed or misplaced block breaks the rotation mode);
  * shuffling the element order leaves the summed K unchanged;
  * the scatter map points at (dof_a, dof_b) and the block rank map at the
    node position in the sorted adjacency;
  * supports: constrained rows/columns zero except the kept diagonal.
"""
import itertools

import numpy as np
import pytest

import workloads as W
from oracle import assembly as A


def mixed_problem():
    P = W.tiny_shell(2, seed=1)
    # add two beams along the first grid line (nodes 0-1, 1-2) -> mixed mesh
    P["beam_conn"] = np.array([[0, 1], [1, 2]], np.int32)
    P["A"] = np.full(2, 1e-3)
    P["Iy"] = np.full(2, 1e-6)
    P["Iz"] = np.full(2, 2e-6)
    P["J"] = np.full(2, 2e-6)
    P["E"] = np.concatenate([np.full(2, 210e9), P["E"]])
    P["nu"] = np.concatenate([np.full(2, 0.3), P["nu"]])
    return P


PROBLEMS = {
    "beam": lambda: W.tiny_beam_grid(0),
    "shell3": lambda: W.tiny_shell(3, 0),
    "mixed": mixed_problem,
    "C1": W.config1,
}


def brute_pairs(P):
    pairs = set()
    ne = A.n_beams(P) + A.n_quads(P)
    for e in range(ne):
        nodes = A.element_nodes(P, e)
        for a, b in itertools.product(nodes, nodes):
            pairs.add((a, b))
    return pairs


@pytest.mark.parametrize("name", list(PROBLEMS))
def test_pattern_brute_force(name):
    P = PROBLEMS[name]()
    nd = 6 * len(P["x"])
    row_ptr, col_idx, vals = A.csr_from_dok(A.assemble_dok(P), nd)
    got = set()
    for r in range(nd):
        for k in range(row_ptr[r], row_ptr[r + 1]):
            got.add((r, int(col_idx[k])))
    want = {(6 * a + ca, 6 * b + cb) for (a, b) in brute_pairs(P) for ca in range(6) for cb in range(6)}
    assert got == want
    # columns strictly ascending within each row
    for r in range(nd):
        seg = col_idx[row_ptr[r]:row_ptr[r + 1]]
        assert np.all(np.diff(seg) > 0)


@pytest.mark.parametrize("n", [1, 2, 3, 5])
def test_grid_nnz_formula(n):
    P = W.tiny_shell(n, 0)
    row_ptr, _, _ = A.csr_from_dok(A.assemble_dok(P), 6 * (n + 1) ** 2)
    assert row_ptr[-1] == 36 * ((n + 1) ** 2 + 4 * n * (n + 1) + 4 * n * n)


@pytest.mark.parametrize("name", list(PROBLEMS))
def test_global_rigid_modes(name):
    P = PROBLEMS[name]()
    nn = len(P["x"])
    K = A.dense_from_dok(A.assemble_dok(P), 6 * nn)
    X = A.coords(P)
    c = X.mean(axis=0)
    nrm = np.linalg.norm(K)
    for k in range(3):
        r = np.zeros(6 * nn)
        r[k::6] = 1.0
        assert np.linalg.norm(K @ r) <= 1e-12 * nrm * np.linalg.norm(r)
        w = np.zeros(3)
        w[k] = 1.0
        r = np.zeros(6 * nn)
        for i in range(nn):
            r[6 * i:6 * i + 3] = np.cross(w, X[i] - c)
            r[6 * i + 3:6 * i + 6] = w
        assert np.linalg.norm(K @ r) <= 1e-12 * nrm * np.linalg.norm(r)


def test_shuffle_invariance():
    P = mixed_problem()
    nd = 6 * len(P["x"])
    ne = A.n_beams(P) + A.n_quads(P)
    K0 = A.dense_from_dok(A.assemble_dok(P), nd)
    rng = np.random.default_rng(5)
    order = rng.permutation(ne)
    K1 = A.dense_from_dok(A.assemble_dok(P, order=order), nd)
    assert np.abs(K1 - K0).max() <= 1e-15 * np.abs(K0).max() * 4


def test_scatter_and_rank_maps():
    P = mixed_problem()
    nd = 6 * len(P["x"])
    row_ptr, col_idx, _ = A.csr_from_dok(A.assemble_dok(P), nd)
    pos = A.scatter_map(P, row_ptr, col_idx)
    adj = A.node_adjacency(P)
    rank = A.block_rank(P)
    ne = A.n_beams(P) + A.n_quads(P)
    for e in range(ne):
        nodes = A.element_nodes(P, e)
        dofs = A.element_dofs(nodes)
        for a, ra in enumerate(dofs):
            for b, cb in enumerate(dofs):
                k = pos[e][a, b]
                assert row_ptr[ra] <= k < row_ptr[ra + 1] and col_idx[k] == cb
        k = len(nodes)
        for i in range(k):
            for j in range(k):
                assert adj[nodes[i]][rank[e][i * k + j]] == nodes[j]


def test_supports_elimination():
    P = W.tiny_shell(2, 3)
    nd = 6 * len(P["x"])
    dok = A.assemble_dok(P)
    K = A.dense_from_dok(dok, nd)
    fixed = A.fixed_dofs(P)
    assert fixed.sum() == 12
    Kb, fb = A.apply_supports_dense(K, P["f"], fixed)
    for c in np.nonzero(fixed)[0]:
        assert Kb[c, c] == K[c, c]
        assert np.count_nonzero(Kb[c]) == 1 and np.count_nonzero(Kb[:, c]) == 1
        assert fb[c] == 0.0
    free = ~fixed
    assert np.array_equal(Kb[np.ix_(free, free)], K[np.ix_(free, free)])
    # CSR form agrees with the dense form
    row_ptr, col_idx, vals = A.csr_from_dok(dok, nd)
    v2 = A.apply_supports_csr(row_ptr, col_idx, vals, fixed)
    Kd = np.zeros((nd, nd))
    for r in range(nd):
        for k in range(row_ptr[r], row_ptr[r + 1]):
            Kd[r, col_idx[k]] = v2[k]
    assert np.array_equal(Kd, Kb)


@pytest.mark.parametrize("name", ["shell3", "mixed"])
def test_node_rows_equal_dok(name):
    P = PROBLEMS[name]()
    nd = 6 * len(P["x"])
    K = A.dense_from_dok(A.assemble_dok(P), nd)
    for n in range(len(P["x"])):
        rows = A.node_rows(P, n)
        got = np.zeros((6, nd))
        for col, v in rows.items():
            got[:, col] = v
        assert np.abs(got - K[6 * n:6 * n + 6]).max() <= 1e-15 * np.abs(K).max() * 4
        assert set(rows) == set(np.nonzero(np.any(K[6 * n:6 * n + 6] != 0, axis=0))[0]) | set(rows)
