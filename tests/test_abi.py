"""CPU-only checks of the C-ABI library: it loads, exports every symbol that
include/sso.h declares, and its host-side validation returns the documented
error codes without touching a GPU."""
import ctypes as C
import os
import re

import numpy as np
import pytest

import workloads as W

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    src = open(os.path.join(ROOT, "include", "sso.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(sso_[A-Za-z_]+)\s*\(", src)))


def test_library_exports_every_header_symbol():
    import paper_2407_20026_b200 as sso
    lib = C.CDLL(sso.LIB_PATH)
    syms = header_symbols()
    assert len(syms) >= 20
    for s in syms:
        assert hasattr(lib, s), s
    assert set(syms) == set(sso.EXPORTED)


def test_library_is_sm100a():
    import paper_2407_20026_b200 as sso
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", sso.LIB_PATH], capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout


def _expect(P, code, **kw):
    import paper_2407_20026_b200 as sso
    with pytest.raises(sso.SSOError) as ei:
        sso.Model(P, **kw)
    assert ei.value.code == code, str(ei.value)
    return str(ei.value)


def test_validation_errors():
    import paper_2407_20026_b200.api as A
    P = W.tiny_shell(2, 0)
    Q = dict(P, quad_conn=P["quad_conn"].copy())
    Q["quad_conn"][1, 2] = 999
    assert "out of range" in _expect(Q, A.SSO_E_INVALID)
    Q = dict(P, quad_conn=P["quad_conn"].copy())
    Q["quad_conn"][0, 1] = Q["quad_conn"][0, 0]
    assert "repeated node" in _expect(Q, A.SSO_E_INVALID)
    _expect(dict(P, t=-P["t"]), A.SSO_E_INVALID)
    _expect(dict(P, E=np.zeros_like(P["E"])), A.SSO_E_INVALID)
    _expect(dict(P, nu=np.full_like(P["nu"], 0.5)), A.SSO_E_INVALID)
    _expect(dict(P, sup_node=np.zeros(0, np.int32), sup_mask=np.zeros(0, np.uint8)), A.SSO_E_INVALID)
    _expect(dict(P, sup_mask=np.zeros_like(P["sup_mask"])), A.SSO_E_INVALID)
    x = P["x"].copy()
    x[3] = np.nan
    _expect(dict(P, x=x), A.SSO_E_INVALID)
    B = W.tiny_beam_grid(0)
    Bc = dict(B, beam_conn=B["beam_conn"].copy())
    Bc["beam_conn"][0, 1] = Bc["beam_conn"][0, 0]
    assert "i_node == j_node" in _expect(Bc, A.SSO_E_INVALID)
    Bz = dict(B, x=B["x"].copy(), y=B["y"].copy(), z=B["z"].copy())
    a, b = Bz["beam_conn"][0]
    Bz["x"][b], Bz["y"][b], Bz["z"][b] = Bz["x"][a], Bz["y"][a], Bz["z"][a]
    assert "zero length" in _expect(Bz, A.SSO_E_DEGENERATE)
    _expect(dict(B, Iy=np.zeros_like(B["Iy"])), A.SSO_E_INVALID)
    _expect(P, A.SSO_E_INVALID, rtol=-1.0)


def test_no_gpu_reports_cuda_error():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import paper_2407_20026_b200.api as A
    _expect(W.tiny_shell(2, 0), A.SSO_E_CUDA)


def test_nccl_resolves_at_run_time():
    """The strips' NCCL transport is resolved with dlopen (no link-time dependency): the
    library finds libnccl.so.2 in this environment and forms a unique id (bootstrap only, no
    GPU needed) -- what bench.py --gpus N broadcasts before creating the rank handles."""
    import torch  # noqa: F401  (the process's libnccl.so.2, as under torchrun)
    import paper_2407_20026_b200 as sso
    uid = sso.nccl_unique_id()
    assert isinstance(uid, bytes) and len(uid) == 128 and any(uid)
