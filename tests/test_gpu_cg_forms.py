"""GPU parity of the CG loop forms (reading c5):

  * the fused x / r / p update (cg_update_fused_kernel, ping-pong p buffers, one grid
    barrier) against the classic update + p-update kernels (SSO_CG_FUSED=0);
  * the same for the node-block Jacobi preconditioner (precond = 1,
    cg_update_block_fused_kernel / cg_pfix_z_kernel);
  * the reliable-update modes 0 (recurrence only), 1 (final true-residual check and
    restart, the default) and 2 (also periodic residual replacement, which re-forms p
    from the previous p buffer in the fused form: cg_pfix_kernel).

Each solve is checked against the oracle's Cholesky solution (|u - u_ref| <= 1e-9
|u_ref|, the tolerance of tests/test_gpu_parity.py); the mid-size grid, whose oracle
solve would be slow, is checked for its true residual and against the classic form.
"""
import os

import numpy as np
import pytest

import workloads as W
from oracle import grad as OG

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def sso():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a B200"
    import paper_2407_20026_b200 as m
    return m


def _model(sso, P, fused, **kw):
    old = os.environ.get("SSO_CG_FUSED")
    os.environ["SSO_CG_FUSED"] = "1" if fused else "0"
    try:
        return sso.Model(P, **kw)
    finally:
        if old is None:
            del os.environ["SSO_CG_FUSED"]
        else:
            os.environ["SSO_CG_FUSED"] = old


@pytest.mark.parametrize("precond", [0, 1])
@pytest.mark.parametrize("storage", [1, 3])
@pytest.mark.parametrize("reliable", [0, 1, 2])
@pytest.mark.parametrize("fused", [False, True])
@pytest.mark.parametrize("make", [W.config1, W.config2])
def test_cg_forms_against_oracle(sso, make, fused, reliable, storage, precond):
    P = make()
    m = _model(sso, P, fused, rtol=1e-12, reliable=reliable, storage=storage, precond=precond, check_every=8)
    m.assemble()
    u, info = m.solve(P["f"])
    assert info["status"] == 0
    uref, _, _ = OG.evaluate(P)
    assert np.linalg.norm(u - uref) <= 1e-9 * np.linalg.norm(uref)


@pytest.mark.parametrize("precond", [0, 1])
@pytest.mark.parametrize("reliable", [1, 2])
def test_fused_matches_classic_midsize(sso, reliable, precond):
    """80 x 80 shell (39 366 DOF, hundreds of iterations over many chunks, periodic
    replacements with reliable = 2): fused and classic forms reach the same solution."""
    P = W.shell_config3(80, cfg=3)
    out = {}
    for fused in (False, True):
        m = _model(sso, P, fused, rtol=1e-11, reliable=reliable, precond=precond)
        m.assemble()
        u, info = m.solve(P["f"])
        assert info["status"] == 0 and info["true_rel_res"] < 1e-10
        out[fused] = (u, info["iters"])
    (u0, i0), (u1, i1) = out[False], out[True]
    assert np.linalg.norm(u1 - u0) <= 1e-9 * np.linalg.norm(u0)
    assert abs(i1 - i0) <= max(3, i0 // 100)


@pytest.mark.parametrize("precond", [0, 1])
@pytest.mark.parametrize("reliable", [1, 2])
def test_fused_batched_designs(sso, reliable, precond):
    """A batch of designs (one CTA set, reduction and grid barrier per design) in the
    fused form equals the classic form design by design."""
    B = 6
    designs = [W.config5_design(b, n=12) for b in range(B)]
    Z = np.stack([d["z"] for d in designs])
    T = np.stack([d["t"] for d in designs])
    F = np.stack([d["f"] for d in designs])
    out = {}
    for fused in (False, True):
        m = _model(sso, designs[0], fused, rtol=1e-12, batch=B, reliable=reliable, precond=precond,
                   check_every=8)
        m.set_design(z=Z, t=T)
        m.assemble()
        U, infos = m.solve(F)
        assert all(i["status"] == 0 for i in infos)
        out[fused] = U
    for b in range(B):
        assert np.linalg.norm(out[True][b] - out[False][b]) <= 1e-9 * np.linalg.norm(out[False][b])
    uref, _, _ = OG.evaluate(designs[2])
    assert np.linalg.norm(out[True][2] - uref) <= 1e-9 * np.linalg.norm(uref)


@pytest.mark.parametrize("precond", [0, 1])
def test_fused_reductions_deterministic(sso, precond):
    """The fused update's all-CTA all-reduce and the SpMV partials summed in every CTA give
    bit-identical iterates: a 200 x 200 shell (242 406 DOF, the full co-resident grid) solved
    twice on one handle and once on a fresh handle returns the same u and iteration count."""
    P = W.shell_config3(200, cfg=3)
    m = sso.Model(P, rtol=1e-8, precond=precond)
    m.assemble()
    u1, i1 = m.solve(P["f"])
    u2, i2 = m.solve(P["f"])
    m3 = sso.Model(P, rtol=1e-8, precond=precond)
    m3.assemble()
    u3, i3 = m3.solve(P["f"])
    assert i1["status"] == 0 and i1["iters"] == i2["iters"] == i3["iters"]
    assert np.array_equal(u1, u2) and np.array_equal(u1, u3)
    assert i1["true_rel_res"] < 1e-7
