"""GPU parity of the partitioned (multi-strip) path, SURVEY.md §8(e).

P contiguous node strips held by one handle on one GPU (in-process transport:
device-to-device halo copies and a fixed-order allreduce of the CG scalars)
run exactly the distributed algorithm the NCCL transport runs across GPUs:
the single-reduction CG of csrc/cg_sr.cu (halo exchange of u = M^-1 r and ONE
allreduce of (u^T K u, r^T u, r^T r) per iteration), optionally with the interior
rows' SpMV overlapping the halo exchange (SSO_SPLIT=1: row ranges of the pull
SpMV, side stream), halo of u before the gradient, owned-slice outputs.  Checked
against the single-strip handle and the oracle:

  * strip-local assembled values concatenate to the global CSR bit-exactly;
  * u within 1e-9 of the oracle (Cholesky), C within 1e-10, gradients 1e-7;
  * CG iteration counts within 2 of the single-strip run (only the order of
    the dot-product sums differs).
"""
import numpy as np
import pytest

import workloads as W
from _tol import assert_components
from oracle import grad as OG

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def sso():
    import torch
    assert torch.cuda.is_available()
    import paper_2407_20026_b200 as m
    return m


def mixed():
    P = W.tiny_shell(4, seed=3)
    P["beam_conn"] = np.array([[0, 6], [6, 12], [3, 9], [20, 24]], np.int32)
    nb = len(P["beam_conn"])
    P["A"], P["Iy"], P["Iz"], P["J"] = (np.full(nb, 1e-3), np.full(nb, 2e-6), np.full(nb, 1e-6),
                                        np.full(nb, 2e-6))
    P["E"] = np.concatenate([np.full(nb, 210e9), P["E"]])
    P["nu"] = np.concatenate([np.full(nb, 0.3), P["nu"]])
    return P


CASES = [
    ("C2", W.config2, 2, None),
    ("C2", W.config2, 3, [0, 40, 300, 441]),
    ("C2", W.config2, 4, None),
    ("mixed", mixed, 3, None),
    ("C1", W.config1, 2, None),
]


@pytest.mark.parametrize("storage", [1, 3])
@pytest.mark.parametrize("name,make,nparts,ranges", CASES)
def test_partitioned_matches_single_and_oracle(sso, name, make, nparts, ranges, storage):
    P = make()
    # same storage on one strip and on P strips: full rows are formed by the same kernels in
    # the same element order (bit-comparable); with upper blocks (storage 3) a block across a
    # strip edge is stored by its local-order lower endpoint (owned before halo), which can be
    # the other endpoint than in the global order -> equal to rounding
    m1 = sso.Model(P, rtol=1e-12, storage=storage)
    m1.assemble()
    mp = sso.Model(P, rtol=1e-12, n_parts=nparts, part_ranges=ranges, storage=storage)
    assert mp.storage_info()[2] == (3 if storage == 3 else 0)
    assert mp.n_parts_here == nparts
    mp.assemble()
    rp1, ci1, v1 = m1.export_csr()
    rpp, cip, vp = mp.export_csr()
    assert np.array_equal(rp1, rpp) and np.array_equal(ci1, cip)
    if storage == 1:
        assert np.array_equal(v1, vp)
    else:
        for r in range(len(rp1) - 1):
            seg = slice(rp1[r], rp1[r + 1])
            assert np.abs(v1[seg] - vp[seg]).max() <= 1e-14 * np.abs(v1[seg]).max()
    assert np.array_equal(m1.export_dinv(), mp.export_dinv())
    u1, i1 = m1.solve(P["f"])
    up, ip = mp.solve(P["f"])
    assert ip["status"] == 0 and abs(ip["iters"] - i1["iters"]) <= max(2, 0.03 * i1["iters"])
    uref, _, _ = OG.evaluate(P)
    assert np.linalg.norm(up - uref) <= 1e-9 * np.linalg.norm(uref)
    assert np.linalg.norm(up - u1) <= 1e-10 * np.linalg.norm(u1)
    Cp, dXp, dTp = mp.grad()
    C1, dX1, dT1 = m1.grad()
    Cref = OG.compliance(P["f"], uref)
    assert abs(Cp - Cref) <= 1e-10 * abs(Cref)
    # gradients at the same seeded state: partitioned == single strip
    u = W.random_state(len(P["x"]), 5)
    C1s, dX1s, dT1s = m1.grad_at(P["f"], u)
    Cps, dXps, dTps = mp.grad_at(P["f"], u)
    assert np.array_equal(dX1s, dXps)
    assert np.array_equal(dT1s, dTps)
    assert Cps == pytest.approx(C1s, rel=1e-13)
    # and at the solved state vs the oracle's adjoint gradient
    gX, gT = OG.adjoint_gradient(P, uref, 1.0)
    assert_components(dXp, gX, 1e-7, "partitioned dC/dX")
    # spmv through the halo exchange
    x = np.random.default_rng(1).standard_normal(6 * len(P["x"]))
    assert np.allclose(mp.spmv(x), m1.spmv(x), rtol=0, atol=1e-12 * np.abs(m1.spmv(x)).max())


@pytest.mark.parametrize("split", ["0", "1"])
@pytest.mark.parametrize("precond", [0, 1])
def test_partitioned_c3_family_iterations(sso, split, precond, monkeypatch):
    """A 60x60 C3-recipe shell (clamped edges) in 4 strips: same solution and iteration count
    (within 1 %) as one strip, with and without the interior / boundary split of the SpMV
    (which also takes the row-range pieces of the pull kernel and the side-stream halo), and
    the certification fields consistent with the single strip's."""
    monkeypatch.setenv("SSO_SPLIT", split)
    P = W.shell_config3(60, cfg=3)
    m1 = sso.Model(P, rtol=1e-10, precond=precond)
    m1.assemble()
    m4 = sso.Model(P, rtol=1e-10, n_parts=4, precond=precond)
    m4.assemble()
    u1, i1 = m1.solve(P["f"])
    u4, i4 = m4.solve(P["f"])
    # same algorithm in exact arithmetic; the dot products are summed in another order (per
    # strip, and per SpMV piece with the split), which moves the count by a few iterations
    assert i4["status"] == 0 and abs(i1["iters"] - i4["iters"]) <= max(3, 0.01 * i1["iters"])
    d = np.linalg.norm(u4 - u1) / np.linalg.norm(u1)
    assert d <= 1e-8 and d <= 1.01 * (i1["err2_est"] + i4["err2_est"]) + 1e-14
    assert i4["lanczos_lmax"] == pytest.approx(i1["lanczos_lmax"], rel=1e-6)
    assert i4["lanczos_lmin"] == pytest.approx(i1["lanczos_lmin"], rel=1e-3)
    C1, dX1, dT1 = m1.grad()
    C4, dX4, dT4 = m4.grad()
    assert C4 == pytest.approx(C1, rel=1e-9)
    assert_components(dX4, dX1, 1e-7, "dC/dX 4 strips vs 1")


def test_batched_designs_match_single(sso):
    """C5-style batch: B designs sharing connectivity run in the same
    kernels with their own CG scalars; each equals an independent single-design run."""
    B = 5
    designs = [W.config5_design(b, n=20) for b in range(B)]
    P0 = designs[0]
    mb = sso.Model(P0, rtol=1e-12, batch=B)
    mb.set_design(z=np.stack([d["z"] for d in designs]), t=np.stack([d["t"] for d in designs]))
    mb.assemble()
    F = np.stack([d["f"] for d in designs])
    U, infos = mb.solve(F)
    Cb, dXb, dTb = mb.grad()
    Ug = W.random_state(len(P0["x"]), 3)
    Cg, dXg, dTg = mb.grad_at(F, np.stack([Ug] * B))
    for b, d in enumerate(designs):
        m1 = sso.Model(d, rtol=1e-12)
        m1.assemble()
        u1, i1 = m1.solve(d["f"])
        assert infos[b]["status"] == 0
        # same algorithm per design; only the reduction partition differs
        assert abs(infos[b]["iters"] - i1["iters"]) <= max(2, 0.15 * i1["iters"])
        assert np.linalg.norm(U[b] - u1) <= 1e-9 * np.linalg.norm(u1)
        C1, dX1, dT1 = m1.grad()
        assert Cb[b] == pytest.approx(C1, rel=1e-10)
        C1g, dX1g, dT1g = m1.grad_at(d["f"], Ug)
        assert np.array_equal(dXg[b], dX1g) and np.array_equal(dTg[b], dT1g)
    uref, _, _ = OG.evaluate(designs[2])
    assert np.linalg.norm(U[2] - uref) <= 1e-9 * np.linalg.norm(uref)


@pytest.mark.parametrize("nparts", [5, 11])
def test_split_thin_strips(sso, nparts, monkeypatch):
    """Strips of one or two node rows have no interior rows: every SpMV piece of the
    interior/boundary split is a boundary piece (or empty), and the u^T K u pieces must still
    start from zero each iteration."""
    monkeypatch.setenv("SSO_SPLIT", "1")
    P = W.shell_config3(10, cfg=3)
    m1 = sso.Model(P, rtol=1e-12)
    m1.assemble()
    mp = sso.Model(P, rtol=1e-12, n_parts=nparts)
    mp.assemble()
    u1, i1 = m1.solve(P["f"])
    up, ip = mp.solve(P["f"])
    assert ip["status"] == 0 and abs(ip["iters"] - i1["iters"]) <= max(3, 0.01 * i1["iters"])
    assert np.linalg.norm(up - u1) <= 1e-9 * np.linalg.norm(u1)


@pytest.mark.parametrize("precond", [0, 1])
@pytest.mark.parametrize("make", [W.config2, lambda: W.shell_config3(40, cfg=3)])
def test_nccl_transport_single_rank(sso, make, precond, monkeypatch):
    """The NCCL transport of the strips on ONE rank (SSO_NCCL_SELF=1: a 1-rank communicator, no
    peer to wait for): comm init from a unique id, the halo group (empty) and the allreduces of
    the single-reduction CG inside the captured graphs, the interior / boundary split on the
    side stream -- the code a multi-GPU run executes, here against the local single-part solve."""
    P = make()
    monkeypatch.setenv("SSO_NCCL_SELF", "1")
    m = sso.Model(P, rtol=1e-12, nranks=1, rank=0, nccl_id=sso.nccl_unique_id(), precond=precond)
    m.assemble()
    u, info = m.solve(P["f"])
    C, dX, dT = m.grad()
    m.close()
    monkeypatch.delenv("SSO_NCCL_SELF")
    m0 = sso.Model(P, rtol=1e-12, precond=precond)
    m0.assemble()
    u0, info0 = m0.solve(P["f"])
    C0, dX0, dT0 = m0.grad()
    m0.close()
    assert info["status"] == 0 and info["true_rel_res"] < 1e-11
    assert np.linalg.norm(u - u0) <= 1e-10 * np.linalg.norm(u0)
    assert C == pytest.approx(C0, rel=1e-10)
    assert np.max(np.abs(dX - dX0)) <= 1e-8 * np.max(np.abs(dX0))
    assert np.max(np.abs(dT - dT0)) <= 1e-8 * np.max(np.abs(dT0))
    assert abs(info["iters"] - info0["iters"]) <= max(3, info0["iters"] // 50)
