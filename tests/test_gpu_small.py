"""GPU parity of the cluster-resident small-model PCG (csrc/cg_small.cu).

Models up to 1 152 nodes (one thread-block cluster of <= 16 CTAs per design) run their CG
chunks in cg_cluster_kernel.  Checked here against the oracle and against the two-kernel
fused path (SSO_SMALL=0) of the same library:
  * C1 (beams, a single CTA) and C2 (a 16-CTA cluster): u against the oracle's Cholesky
    solution, the same iteration count and Lanczos extremes as the fused path;
  * a 30 x 30 shell (961 nodes, the largest cluster shape) against the oracle;
  * a batch of designs (one cluster per design) against single-design solves;
  * a 34 x 34 shell (1 225 nodes, beyond one cluster) still solves (the fused path).
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


def _model(sso, P, small, **kw):
    old = os.environ.get("SSO_SMALL")
    os.environ["SSO_SMALL"] = "1" if small else "0"
    try:
        return sso.Model(P, **kw)
    finally:
        if old is None:
            del os.environ["SSO_SMALL"]
        else:
            os.environ["SSO_SMALL"] = old


def _solve(sso, P, small, **kw):
    m = _model(sso, P, small, **kw)
    m.assemble()
    u, info = m.solve(P["f"])
    C, dX, dT = m.grad()
    m.close()
    return u, info, C, dX


@pytest.mark.parametrize("make", [W.config1, W.config2])
def test_cluster_pcg_matches_oracle_and_fused(sso, make):
    P = make()
    u, info, C, dX = _solve(sso, P, True, rtol=1e-12)
    u0, info0, C0, dX0 = _solve(sso, P, False, rtol=1e-12)
    assert info["status"] == 0 and info["true_rel_res"] < 1e-11
    uref, _, _ = OG.evaluate(P)
    assert np.linalg.norm(u - uref) <= 1e-9 * np.linalg.norm(uref)
    assert np.linalg.norm(u - u0) <= 1e-10 * np.linalg.norm(u0)
    assert abs(info["iters"] - info0["iters"]) <= 2
    assert C == pytest.approx(C0, rel=1e-10)
    assert info["lanczos_iters"] > 0
    # (lambda_min of a Lanczos run is sensitive to the rounding of the recurrence)
    assert info["lanczos_lmin"] == pytest.approx(info0["lanczos_lmin"], rel=1e-4)
    assert info["lanczos_lmax"] == pytest.approx(info0["lanczos_lmax"], rel=1e-6)


def test_cluster_pcg_largest_cluster_shape(sso):
    P = W.shell_config3(30, cfg=3)  # 961 nodes: 16 CTAs of 61 nodes
    u, info, C, dX = _solve(sso, P, True, rtol=1e-12)
    assert info["status"] == 0
    uref, _, _ = OG.evaluate(P)
    assert np.linalg.norm(u - uref) <= 1e-9 * np.linalg.norm(uref)


def test_cluster_pcg_batch(sso):
    """One cluster per design of a batch: every design equals its own single solve."""
    B = 3
    designs = [W.config5_design(b, n=20) for b in range(B)]
    F = np.stack([d["f"] for d in designs])
    m = _model(sso, designs[0], True, rtol=1e-12, batch=B)
    m.set_design(z=np.stack([d["z"] for d in designs]), t=np.stack([d["t"] for d in designs]))
    m.assemble()
    U, infos = m.solve(F)
    Cb = m.grad()[0]
    m.close()
    for b in range(B):
        assert infos[b]["status"] == 0
        u1, info1, C1, _ = _solve(sso, designs[b], True, rtol=1e-12)
        assert np.linalg.norm(U[b] - u1) <= 1e-10 * np.linalg.norm(u1)
        assert Cb[b] == pytest.approx(C1, rel=1e-10)


def test_beyond_one_cluster_uses_the_fused_path(sso):
    P = W.shell_config3(34, cfg=3)  # 1 225 nodes
    u, info, C, dX = _solve(sso, P, True, rtol=1e-10)
    u0, info0, C0, dX0 = _solve(sso, P, False, rtol=1e-10)
    assert info["status"] == 0 and info["iters"] == info0["iters"]
    assert np.array_equal(u, u0)  # the same kernels ran


def test_cluster_pcg_deterministic(sso):
    """Fixed-order reductions: repeated solves (and a second handle) give bit-identical u."""
    P = W.config2()
    u1, i1, C1, dX1 = _solve(sso, P, True, rtol=1e-10)
    u2, i2, C2, dX2 = _solve(sso, P, True, rtol=1e-10)
    m = _model(sso, P, True, rtol=1e-10)
    m.assemble()
    u3, i3 = m.solve(P["f"])
    u4, i4 = m.solve(P["f"])
    m.close()
    assert np.array_equal(u1, u2) and np.array_equal(u1, u3) and np.array_equal(u3, u4)
    assert i1["iters"] == i2["iters"] == i3["iters"] == i4["iters"]
    assert C1 == C2 and np.array_equal(dX1, dX2)
