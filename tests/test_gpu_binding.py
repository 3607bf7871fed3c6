"""Binding checks on the GPU (include/sso.h sso_set_stream; api.py argument checks).

* Stream ordering: device buffers written by torch on its default (legacy) stream right
  before a library call are seen by that call (the handle's stream waits on the legacy
  stream at every entry point), and the library's outputs are complete for torch kernels
  queued after the call.
* Argument checks: wrong dtype, too few elements, non-contiguous tensors and mixed
  host/device buffers raise ValueError before any pointer reaches the library.
"""
import numpy as np
import pytest

import workloads as W

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def sso():
    import paper_2407_20026_b200 as m
    return m


def test_default_stream_ordering(sso):
    import torch
    P = W.config2()
    m = sso.Model(P, rtol=1e-12, device=0)
    m.assemble()
    f0 = torch.from_numpy(P["f"]).cuda()
    u_ref, _ = m.solve(f0.clone())
    u_ref = u_ref.clone()
    for k in range(3):
        f = f0.clone()
        torch.cuda.synchronize()
        torch.cuda._sleep(50_000_000)      # ~25 ms of GPU time on the default stream
        f.mul_(2.0 ** (k + 1))             # queued behind the sleep
        u, info = m.solve(f)               # must see the scaled f
        v = u * 1.0                        # torch kernel right after the call
        assert info["status"] == 0
        assert torch.allclose(v, u_ref * 2.0 ** (k + 1), rtol=1e-8, atol=0)
    # a gradient into caller tensors written just before by torch
    C = torch.full((1,), 7.0, dtype=torch.float64, device="cuda")
    dX = torch.full((3 * m.n_nodes,), 7.0, dtype=torch.float64, device="cuda")
    dT = torch.full((m.n_quads,), 7.0, dtype=torch.float64, device="cuda")
    u, _ = m.solve(f0.clone())
    torch.cuda._sleep(50_000_000)
    C.zero_()
    m.grad(out=(C, dX, dT))
    Cn, dXn, dTn = m.grad()
    assert float(C[0]) == float(Cn)


def test_argument_checks(sso):
    import torch
    P = W.config2()
    m = sso.Model(P, rtol=1e-10, device=0)
    m.assemble()
    f = torch.from_numpy(P["f"]).cuda()
    with pytest.raises(ValueError):
        m.solve(f.float())                                   # wrong dtype
    with pytest.raises(ValueError):
        m.solve(f[: m.ndof // 2])                            # too few elements
    with pytest.raises(ValueError):
        m.solve(torch.stack([f, f], 1)[:, 0])                # non-contiguous
    with pytest.raises(ValueError):
        m.solve(f, u=np.zeros(m.ndof))                       # mixed host / device
    with pytest.raises(ValueError):
        m.solve(P["f"], u=np.zeros(m.ndof, np.float32))      # host float32 output
    with pytest.raises(ValueError):
        m.spmv(np.zeros(m.ndof - 6))
    u, info = m.solve(f)                                     # the handle still works
    assert info["status"] == 0
