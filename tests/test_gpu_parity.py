"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle on the
same seeded inputs (SURVEY.md §8(c) C8 tolerances, BASELINE.json north_star):

  pattern / indices   bit-exact
  K_e                 |dK_e|_F <= 1e-13 |K_e|_F
  CSR values          |dv| <= 1e-13 max|row|
  u                   |u - u_ref|_2 <= 1e-9 |u_ref|_2
  C                   |dC| <= 1e-10 |C|
  gradients           |dg_i| <= 1e-7 max(|g_ref,i|, 1e-3 |g_ref|_inf)

Sizes span several CTAs with ragged tails (8 quads / 32 beams per element
CTA; 8 nodes per SpMV CTA).
"""
import numpy as np
import pytest

import workloads as W
from _tol import assert_components
from oracle import assembly as OA, grad as OG

pytestmark = pytest.mark.gpu

TOL_KE, TOL_VAL, TOL_U, TOL_C, TOL_G = 1e-13, 1e-13, 1e-9, 1e-10, 1e-7


@pytest.fixture(scope="module")
def sso():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a B200"
    import paper_2407_20026_b200 as m
    return m


def ragged_shell(nx=7, ny=5, seed=3):
    """Non-square ragged grid (35 quads: 4 full element CTAs + a tail of 3)."""
    rng = np.random.default_rng(seed)
    L = 3.0
    xs = np.arange(nx + 1) * L / nx
    ys = np.arange(ny + 1) * L / ny
    x = np.tile(xs, ny + 1)
    y = np.repeat(ys, nx + 1)
    z = 0.4 * np.sin(x) * np.cos(y) + rng.uniform(-0.02, 0.02, x.size)
    conn = []
    for j in range(ny):
        for i in range(nx):
            a = j * (nx + 1) + i
            conn.append([a, a + 1, a + nx + 2, a + nx + 1])
    conn = np.array(conn, np.int32)
    nq = len(conn)
    f = rng.uniform(-1e3, 1e3, 6 * x.size)
    sn = [k for k in range(x.size) if y[k] == 0.0]
    return W._problem("ragged", x, y, z, quad_conn=conn, t=rng.uniform(0.05, 0.2, nq),
                      E=np.full(nq, 30e9), nu=np.full(nq, 0.2), sup_node=sn,
                      sup_mask=[W.CLAMPED] * len(sn), f=f)


def mixed():
    P = W.tiny_shell(3, seed=7)
    P["beam_conn"] = np.array([[0, 1], [1, 2], [2, 3], [0, 4], [4, 8]], np.int32)
    nb = 5
    P["A"], P["Iy"], P["Iz"], P["J"] = (np.full(nb, 1e-3), np.full(nb, 2e-6), np.full(nb, 1e-6),
                                        np.full(nb, 2e-6))
    P["E"] = np.concatenate([np.full(nb, 210e9), P["E"]])
    P["nu"] = np.concatenate([np.full(nb, 0.3), P["nu"]])
    return P


PROBLEMS = {
    "C1": W.config1,
    "C2": W.config2,
    "tiny2": lambda: W.tiny_shell(2, 0),
    "tiny3edge": lambda: W.tiny_shell(3, 1, supports="edge"),
    "beamgrid": lambda: W.tiny_beam_grid(0),
    "ragged": ragged_shell,
    "mixed": mixed,
}


@pytest.fixture(scope="module")
def cases():
    return {}


def oracle_case(cases, name):
    if name not in cases:
        P = PROBLEMS[name]()
        nd = 6 * len(P["x"])
        dok = OA.assemble_dok(P)
        rp, ci, v = OA.csr_from_dok(dok, nd)
        fixed = OA.fixed_dofs(P)
        vbc = OA.apply_supports_csr(rp, ci, v, fixed)
        u, Kb, fb = OG.evaluate(P, "cholesky")
        cases[name] = dict(P=P, rp=rp, ci=ci, v=v, vbc=vbc, u=u, fixed=fixed)
    return cases[name]


@pytest.mark.parametrize("name", list(PROBLEMS))
def test_pattern_bit_exact(sso, cases, name):
    c = oracle_case(cases, name)
    m = sso.Model(c["P"])
    rp, ci, _ = m.export_csr(values=False)
    assert np.array_equal(rp, c["rp"])
    assert np.array_equal(ci, c["ci"])
    assert np.array_equal(m.export_scatter(), np.concatenate(
        [np.asarray(r, np.int32) for r in OA.block_rank(c["P"])]) if len(OA.block_rank(c["P"])) else [])


@pytest.mark.parametrize("name", list(PROBLEMS))
def test_element_matrices(sso, cases, name):
    c = oracle_case(cases, name)
    P = c["P"]
    m = sso.Model(P)
    m.assemble()
    nb, nq = len(P["beam_conn"]), len(P["quad_conn"])
    for first, count in ((0, nb), (nb, nq)):
        if count == 0:
            continue
        ke = m.export_ke(first, count)
        for k in range(count):
            ref = OA.element_K(P, first + k)
            assert np.linalg.norm(ke[k] - ref) <= TOL_KE * np.linalg.norm(ref), (first + k)


@pytest.mark.parametrize("name", list(PROBLEMS))
def test_csr_values_with_supports(sso, cases, name):
    c = oracle_case(cases, name)
    m = sso.Model(c["P"])
    m.assemble()
    _, _, v = m.export_csr()
    rp = c["rp"]
    ref = c["vbc"]
    for r in range(len(rp) - 1):
        seg = slice(rp[r], rp[r + 1])
        scale = np.abs(ref[seg]).max()
        assert np.abs(v[seg] - ref[seg]).max() <= TOL_VAL * scale, r
    dinv = m.export_dinv()
    diag = np.array([ref[rp[r] + np.searchsorted(c["ci"][rp[r]:rp[r + 1]], r)] for r in range(len(rp) - 1)])
    assert np.allclose(dinv, 1.0 / diag, rtol=1e-13, atol=0)


@pytest.mark.parametrize("name", list(PROBLEMS))
def test_solve_and_gradient(sso, cases, name):
    c = oracle_case(cases, name)
    P = c["P"]
    m = sso.Model(P, rtol=1e-12)
    m.assemble()
    u, info = m.solve(P["f"])
    assert info["status"] == 0 and info["true_rel_res"] < 1e-11
    uref = c["u"]
    assert np.linalg.norm(u - uref) <= TOL_U * np.linalg.norm(uref)
    for obj, s in ((sso.OBJ_COMPLIANCE, 1.0), (sso.OBJ_STRAIN_ENERGY, 0.5)):
        Cv, dX, dT = m.grad(obj)
        Cref = OG.compliance(P["f"], uref, s)
        assert abs(Cv - Cref) <= TOL_C * abs(Cref)
    # gradient parity at the oracle's own state (grad_at): isolates stage A4 exactly
    Cv, dX, dT = m.grad_at(P["f"], uref, sso.OBJ_COMPLIANCE)
    gX, gT = OG.adjoint_gradient(P, uref, 1.0)
    floor = 1e-3 * np.abs(gX).max()
    assert np.all(np.abs(dX - gX) <= TOL_G * np.maximum(np.abs(gX), floor))
    if len(P["quad_conn"]):
        floor = 1e-3 * np.abs(gT).max()
        assert np.all(np.abs(dT - gT) <= TOL_G * np.maximum(np.abs(gT), floor))
    # and through the solved state
    Cv, dX2, dT2 = m.grad(sso.OBJ_COMPLIANCE)
    assert_components(dX2, gX, TOL_G, "dC/dX through the solve")
    if len(P["quad_conn"]):
        assert_components(dT2, gT, TOL_G, "dC/dt through the solve")


def test_determinism_and_scaling(sso):
    P = W.config2()
    m = sso.Model(P, rtol=1e-12)
    m.assemble()
    u1, i1 = m.solve(P["f"])
    u2, i2 = m.solve(P["f"])
    assert np.array_equal(u1, u2) and i1["iters"] == i2["iters"]
    g1 = m.grad()
    g2 = m.grad()
    assert np.array_equal(g1[1], g2[1]) and np.array_equal(g1[2], g2[2])
    u3, _ = m.solve(2.0 * P["f"])
    assert np.array_equal(u3, 2.0 * u1)
    m2 = sso.Model(dict(P, E=2.0 * P["E"]), rtol=1e-12)
    m2.assemble()
    u4, _ = m2.solve(P["f"])
    assert np.array_equal(u4, 0.5 * u1)


def test_device_pointers_and_warm_start(sso):
    import torch
    P = W.config2()
    m = sso.Model(P, rtol=1e-12)
    m.assemble()
    u_h, info_h = m.solve(P["f"])
    f_d = torch.from_numpy(P["f"]).cuda()
    u_d, info_d = m.solve(f_d)
    assert np.array_equal(u_d.cpu().numpy(), u_h)
    Cd, dXd, dTd = m.grad()
    Ch, dXh, dTh = m.grad_at(P["f"], u_h)
    assert Cd == Ch
    assert np.array_equal(dXd, dXh)
    mw = sso.Model(P, rtol=1e-12, warm_start=True)
    mw.assemble()
    u0 = torch.from_numpy(u_h).cuda().clone()
    u_w, info_w = mw.solve(f_d, u0)
    assert info_w["iters"] <= 2
    assert np.linalg.norm(u_w.cpu().numpy() - u_h) <= 1e-10 * np.linalg.norm(u_h)


def test_numeric_errors(sso):
    import paper_2407_20026_b200.api as A
    # isolated node -> zero diagonal on a free DOF -> SINGULAR naming the node
    P = W.tiny_shell(2, 0)
    Q = dict(P, x=np.append(P["x"], 5.0), y=np.append(P["y"], 5.0), z=np.append(P["z"], 0.0),
             f=np.append(P["f"], np.zeros(6)))
    m = sso.Model(Q)
    with pytest.raises(A.SSOError) as ei:
        m.assemble()
    assert ei.value.code == A.SSO_E_SINGULAR and "node 9" in str(ei.value)
    # degenerate quad via set_design (collapsed element) -> DEGENERATE
    m = sso.Model(P)
    x = P["x"].copy()
    y = P["y"].copy()
    z = P["z"].copy()
    x[4], y[4], z[4] = x[0], y[0], z[0]
    m.set_design(x=x, y=y, z=z)
    with pytest.raises(A.SSOError) as ei:
        m.assemble()
    assert ei.value.code == A.SSO_E_DEGENERATE
    # call order
    m = sso.Model(P)
    with pytest.raises(A.SSOError) as ei:
        m.solve(P["f"])
    assert ei.value.code == A.SSO_E_STATE
    # max_iter -> NOT_CONVERGED with the last iterate returned
    m = sso.Model(W.config2(), max_iter=5, check_every=4)
    m.assemble()
    u, info = m.solve(W.config2()["f"], raise_on_error=False)
    assert info["status"] == A.SSO_E_NOT_CONVERGED and info["iters"] == 5
    # zero load -> u = 0 immediately
    m = sso.Model(P)
    m.assemble()
    u, info = m.solve(np.zeros(m.ndof))
    assert info["iters"] == 0 and not np.any(u)


def test_set_design_matches_fresh_model(sso):
    P = W.config2()
    Q = dict(P, z=P["z"] * 1.1, t=P["t"] * 0.9)
    m = sso.Model(P, rtol=1e-12)
    m.set_design(z=Q["z"], t=Q["t"])
    m.assemble()
    u1, _ = m.solve(P["f"])
    m2 = sso.Model(Q, rtol=1e-12)
    m2.assemble()
    u2, _ = m2.solve(P["f"])
    assert np.array_equal(u1, u2)


@pytest.mark.parametrize("make", [W.config2, ragged_shell, lambda: W.shell_config3(40, cfg=3)])
def test_fused_assembly_matches_staged(sso, make):
    """The fused element+assembly pass (default for quad meshes) and the staged path
    (element kernel + segmented gather) produce the same CSR values and dinv."""
    P = make()
    mf = sso.Model(P, assembly=0)
    ms = sso.Model(P, assembly=1)
    mf.assemble()
    ms.assemble()
    rp, ci, vf = mf.export_csr()
    _, _, vs = ms.export_csr()
    for r in range(len(rp) - 1):
        seg = slice(rp[r], rp[r + 1])
        assert np.abs(vf[seg] - vs[seg]).max() <= 1e-14 * np.abs(vs[seg]).max()
    assert np.allclose(mf.export_dinv(), ms.export_dinv(), rtol=1e-14, atol=0)


@pytest.mark.parametrize("storage", [3])
@pytest.mark.parametrize("make", [W.config2, mixed, W.config1, lambda: W.shell_config3(40, cfg=3)])
def test_symmetric_storage_matches_full(sso, make, storage):
    """Upper-block (symmetric) storage with the one-pass pull SpMV (3) reproduces the
    full-storage operator, solve and gradient."""
    P = make()
    ms = sso.Model(P, rtol=1e-12, storage=storage)
    mf = sso.Model(P, rtol=1e-12, storage=1)
    assert ms.storage_info()[2] and not mf.storage_info()[2]
    assert ms.storage_info()[1] < mf.storage_info()[1]
    ms.assemble()
    mf.assemble()
    rp, ci, vs = ms.export_csr()
    _, _, vf = mf.export_csr()
    for r in range(len(rp) - 1):
        seg = slice(rp[r], rp[r + 1])
        assert np.abs(vs[seg] - vf[seg]).max() <= 1e-14 * np.abs(vf[seg]).max()
    x = np.random.default_rng(4).standard_normal(ms.ndof)
    ys, yf = ms.spmv(x), mf.spmv(x)
    assert np.abs(ys - yf).max() <= 1e-13 * np.abs(yf).max()
    us, i_s = ms.solve(P["f"])
    uf, i_f = mf.solve(P["f"])
    assert np.linalg.norm(us - uf) <= 1e-9 * np.linalg.norm(uf)
    Cs, dXs, _ = ms.grad()
    Cf, dXf, _ = mf.grad()
    assert Cs == pytest.approx(Cf, rel=1e-10)


@pytest.mark.parametrize("make", [lambda: W.tiny_shell(3, 2), lambda: W.tiny_beam_grid(1), W.config1, mixed])
def test_material_gradient_and_set_material(sso, make):
    """SIMP design variable: dC/dE vs the oracle, and
    sso_set_material giving the same state as a fresh model with those moduli."""
    from oracle import grad as OGr
    P = make()
    m = sso.Model(P, rtol=1e-12)
    m.assemble()
    m.solve(P["f"])
    g = m.grad_E()
    uref, _, _ = OG.evaluate(P)
    ref = OGr.material_gradient(P, uref, 1.0)
    fl = 1e-3 * np.abs(ref).max()
    assert np.all(np.abs(g - ref) <= 1e-7 * np.maximum(np.abs(ref), fl))
    C, _, _ = m.grad()
    assert float(np.dot(P["E"], g)) == pytest.approx(-C, rel=1e-9)
    rho = np.random.default_rng(2).uniform(0.2, 1.0, len(P["E"]))
    E2 = P["E"] * rho ** 3
    m.set_material(E2)
    m.assemble()
    u2, _ = m.solve(P["f"])
    G2 = None if P.get("G") is None else P["G"] * rho ** 3
    m2 = sso.Model(dict(P, E=E2, G=G2), rtol=1e-12)
    m2.assemble()
    u3, _ = m2.solve(P["f"])
    assert np.linalg.norm(u2 - u3) <= 1e-12 * np.linalg.norm(u3)


@pytest.mark.parametrize("make", [lambda: W.tiny_shell(3, 4), W.config1, mixed, ragged_shell])
def test_general_objective_adjoint(sso, make):
    """Non-self-adjoint objective g = c^T u: the GPU adjoint solve and
    -lambda^T (dK/dp) u vs the oracle; the primal state survives the adjoint solve."""
    from oracle import grad as OGr
    P = make()
    m = sso.Model(P, rtol=1e-12)
    m.assemble()
    u, _ = m.solve(P["f"])
    fixed = OA.fixed_dofs(P)
    c = np.random.default_rng(6).standard_normal(m.ndof)
    c[fixed] = 0.0
    lam, info = m.adjoint_solve(c)
    assert info["status"] == 0
    uref, Kb, _ = OG.evaluate(P)
    free = np.nonzero(~fixed)[0]
    lref = np.zeros_like(uref)
    lref[free] = np.linalg.solve(Kb[np.ix_(free, free)], c[free])
    assert np.linalg.norm(lam - lref) <= 1e-9 * np.linalg.norm(lref)
    C1, dX1, _ = m.grad()          # primal kept
    assert C1 == pytest.approx(OG.compliance(P["f"], uref), rel=1e-10)
    dX, dT, dE = m.grad_adjoint(lref)
    rX, rT, rE = OGr.adjoint_general(P, uref, lref)
    for got, ref in ((dX, rX), (dE, rE)) + (((dT, rT),) if len(rT) else ()):
        assert_components(got, ref, TOL_G, "general adjoint")


@pytest.mark.parametrize("name", ["C2", "ragged", "mixed", "beamgrid"])
def test_pull_storage_against_oracle(sso, cases, name):
    """Storage 3 (upper blocks, pull SpMV) against the oracle directly: CSR values with
    supports, dinv, u (Cholesky), C and the gradient through the solved state."""
    c = oracle_case(cases, name)
    P = c["P"]
    m = sso.Model(P, rtol=1e-12, storage=3)
    assert m.storage_info()[2] == 3
    m.assemble()
    _, _, v = m.export_csr()
    rp, ref = c["rp"], c["vbc"]
    for r in range(len(rp) - 1):
        seg = slice(rp[r], rp[r + 1])
        assert np.abs(v[seg] - ref[seg]).max() <= TOL_VAL * np.abs(ref[seg]).max(), r
    u, info = m.solve(P["f"])
    assert info["status"] == 0
    uref = c["u"]
    assert np.linalg.norm(u - uref) <= TOL_U * np.linalg.norm(uref)
    Cv, dX, _ = m.grad(sso.OBJ_COMPLIANCE)
    assert abs(Cv - OG.compliance(P["f"], uref)) <= TOL_C * abs(OG.compliance(P["f"], uref))
    gX, _ = OG.adjoint_gradient(P, uref, 1.0)
    assert_components(dX, gX, TOL_G, "dC/dX")


def test_pull_storage_batched(sso):
    """Storage 3 with a batch of designs (grid.y) equals full storage per design."""
    B = 3
    designs = [W.config5_design(b, n=12) for b in range(B)]
    F = np.stack([d["f"] for d in designs])
    out = {}
    for st in (1, 3):
        m = sso.Model(designs[0], rtol=1e-12, batch=B, storage=st)
        m.set_design(z=np.stack([d["z"] for d in designs]), t=np.stack([d["t"] for d in designs]))
        m.assemble()
        U, infos = m.solve(F)
        assert all(i["status"] == 0 for i in infos)
        out[st] = (U, m.grad()[0])
    for b in range(B):
        assert np.linalg.norm(out[3][0][b] - out[1][0][b]) <= 1e-9 * np.linalg.norm(out[1][0][b])
        assert out[3][1][b] == pytest.approx(out[1][1][b], rel=1e-10)


@pytest.mark.parametrize("storage", [1, 3])
@pytest.mark.parametrize("name", ["C2", "ragged", "mixed", "beamgrid", "tiny3edge"])
def test_block_jacobi_against_oracle(sso, cases, name, storage):
    """precond = 1 (node-block Jacobi, reading c19): u equals the oracle's Cholesky u,
    C and the gradient follow, and the iteration count tracks the oracle's block PCG."""
    import scipy.sparse as sps
    from oracle import solve as OS
    c = oracle_case(cases, name)
    P = c["P"]
    m = sso.Model(P, rtol=1e-12, storage=storage, precond=1)
    m.assemble()
    u, info = m.solve(P["f"])
    assert info["status"] == 0 and info["true_rel_res"] < 1e-11
    uref = c["u"]
    assert np.linalg.norm(u - uref) <= TOL_U * np.linalg.norm(uref)
    Cv, dX, _ = m.grad(sso.OBJ_COMPLIANCE)
    Cref = OG.compliance(P["f"], uref)
    assert abs(Cv - Cref) <= TOL_C * abs(Cref)
    nd = 6 * len(P["x"])
    Kb = sps.csr_matrix((c["vbc"], c["ci"], c["rp"]), shape=(nd, nd))
    fb = P["f"].copy()
    fb[list(c["fixed"])] = 0.0
    _, oi = OS.pcg_block(Kb, fb, rtol=1e-12)
    assert abs(info["iters"] - oi["iters"]) <= max(3, 0.05 * oi["iters"])


def test_block_jacobi_batched_and_partitioned(sso):
    """precond = 1 with a batch of designs and with in-process strips equals precond = 1
    single runs (and the oracle)."""
    designs = [W.config5_design(b, n=12) for b in range(3)]
    mb = sso.Model(designs[0], rtol=1e-12, batch=3, precond=1)
    mb.set_design(z=np.stack([d["z"] for d in designs]), t=np.stack([d["t"] for d in designs]))
    mb.assemble()
    U, infos = mb.solve(np.stack([d["f"] for d in designs]))
    for b, d in enumerate(designs):
        uref, _, _ = OG.evaluate(d)
        assert infos[b]["status"] == 0
        assert np.linalg.norm(U[b] - uref) <= TOL_U * np.linalg.norm(uref)
    P = W.config2()
    mp = sso.Model(P, rtol=1e-12, n_parts=3, precond=1)
    mp.assemble()
    up, ip = mp.solve(P["f"])
    m1 = sso.Model(P, rtol=1e-12, precond=1, storage=1)
    m1.assemble()
    u1, i1 = m1.solve(P["f"])
    assert ip["status"] == 0 and abs(ip["iters"] - i1["iters"]) <= 2
    uref, _, _ = OG.evaluate(P)
    assert np.linalg.norm(up - uref) <= TOL_U * np.linalg.norm(uref)
    # point vs block: fewer iterations with the node blocks on a shell
    m0 = sso.Model(P, rtol=1e-12, precond=0)
    m0.assemble()
    _, i0 = m0.solve(P["f"])
    assert i1["iters"] < i0["iters"]
    with pytest.raises(Exception):
        sso.Model(P, storage=2)   # the two-pass transpose layout is retired
    with pytest.raises(Exception):
        sso.Model(P, precond=2)


def test_pull_storage_general_nodes(sso):
    """Nodes beyond the pull kernel's fast path (upper degree > 5 or more than 4 pulled
    blocks) take its general branch: a 4x4 shell with a fan of beams from node 0 to every
    other node of its first two rows, and from those to the last node.  Storage 3 equals
    full storage and the oracle."""
    P = W.tiny_shell(4, seed=9)
    nn = len(P["x"])
    fan = [[0, k] for k in range(2, 10)] + [[k, nn - 1] for k in range(2, 10)]
    P["beam_conn"] = np.array(fan, np.int32)
    nb = len(fan)
    P["A"], P["Iy"], P["Iz"], P["J"] = (np.full(nb, 1e-3), np.full(nb, 2e-6), np.full(nb, 1e-6),
                                        np.full(nb, 2e-6))
    P["E"] = np.concatenate([np.full(nb, 210e9), P["E"]])
    P["nu"] = np.concatenate([np.full(nb, 0.3), P["nu"]])
    m3 = sso.Model(P, rtol=1e-12, storage=3)
    m1 = sso.Model(P, rtol=1e-12, storage=1)
    for m in (m3, m1):
        m.assemble()
    x = np.random.default_rng(2).standard_normal(m3.ndof)
    y3, y1 = m3.spmv(x), m1.spmv(x)
    assert np.abs(y3 - y1).max() <= 1e-13 * np.abs(y1).max()
    u3, i3 = m3.solve(P["f"])
    uref, _, _ = OG.evaluate(P)
    assert i3["status"] == 0
    assert np.linalg.norm(u3 - uref) <= TOL_U * np.linalg.norm(uref)
    C3, _, _ = m3.grad()
    assert abs(C3 - OG.compliance(P["f"], uref)) <= TOL_C * abs(OG.compliance(P["f"], uref))


def test_pull_storage_many_designs(sso):
    """A batch larger than the persistent grid (one CTA per design, many chunks per CTA)
    with the pull SpMV: every design equals its own single-design solve."""
    B = 200
    designs = [W.config5_design(b, n=6) for b in range(B)]
    mb = sso.Model(designs[0], rtol=1e-12, batch=B)
    mb.set_design(z=np.stack([d["z"] for d in designs]), t=np.stack([d["t"] for d in designs]))
    mb.assemble()
    U, infos = mb.solve(np.stack([d["f"] for d in designs]))
    for b in (0, 99, 199):
        m1 = sso.Model(designs[b], rtol=1e-12)
        m1.assemble()
        u1, _ = m1.solve(designs[b]["f"])
        assert infos[b]["status"] == 0
        assert np.linalg.norm(U[b] - u1) <= 1e-9 * np.linalg.norm(u1)


@pytest.mark.parametrize("storage", [1, 3])
@pytest.mark.parametrize("sup", ["corners", "edge"])
def test_single_element(sso, sup, storage):
    """Smallest mesh: one MITC-4 quad (one ragged chunk, one node per CTA slot in use)
    against the oracle -- u, C and the adjoint gradient."""
    P = W.tiny_shell(1, supports=sup)
    m = sso.Model(P, rtol=1e-12, storage=storage)
    m.assemble()
    u, info = m.solve(P["f"])
    assert info["status"] == 0
    uref, _, _ = OG.evaluate(P)
    assert np.linalg.norm(u - uref) <= TOL_U * np.linalg.norm(uref)
    Cv, dX, dT = m.grad(sso.OBJ_COMPLIANCE)
    assert abs(Cv - OG.compliance(P["f"], uref)) <= TOL_C * abs(Cv)
    gX, gT = OG.adjoint_gradient(P, uref, 1.0)
    assert_components(dX, gX, TOL_G, "dC/dX")
    assert_components(dT, gT, TOL_G, "dC/dt")
