"""Thin ctypes binding of the C ABI in include/sso.h (argument marshalling only).

Every step of the hot path runs in the CUDA kernels of libsso.so; this module
only converts numpy arrays / torch tensors to pointers.  There is no CPU
fallback: if libsso.so is missing, importing this module raises.

Names follow include/sso.h: Model.create (sso_create), .assemble, .solve,
.grad, .grad_at, .spmv, .set_design, .export_csr, .export_scatter,
.export_ke, .export_dinv, .profile_*.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libsso.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} not built: run `python -c 'import __graft_entry__ as g; g.build()'`")
_lib = C.CDLL(LIB_PATH)

SSO_OK, SSO_E_INVALID, SSO_E_VALIDATION, SSO_E_NUMERIC = 0, 1, 2, 3
SSO_E_DEGENERATE, SSO_E_SINGULAR, SSO_E_NOT_SPD, SSO_E_NOT_CONVERGED = 11, 31, 32, 33
SSO_E_CUDA, SSO_E_NCCL, SSO_E_OOM, SSO_E_STATE = 40, 41, 42, 43
STATUS_NAMES = {0: "SSO_OK", 1: "SSO_E_INVALID", 2: "SSO_E_VALIDATION", 3: "SSO_E_NUMERIC",
                11: "SSO_E_DEGENERATE", 31: "SSO_E_SINGULAR", 32: "SSO_E_NOT_SPD",
                33: "SSO_E_NOT_CONVERGED", 40: "SSO_E_CUDA", 41: "SSO_E_NCCL", 42: "SSO_E_OOM",
                43: "SSO_E_STATE"}
OBJ_COMPLIANCE, OBJ_STRAIN_ENERGY = 0, 1
MEM_HOST, MEM_DEVICE = 0, 1

_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int32)
_lp = C.POINTER(C.c_int64)
_up = C.POINTER(C.c_uint8)


class sso_mesh(C.Structure):
    _fields_ = [("n_nodes", C.c_int32), ("x", _dp), ("y", _dp), ("z", _dp),
                ("n_beams", C.c_int32), ("beam_conn", _ip), ("n_quads", C.c_int32),
                ("quad_conn", _ip)]


class sso_sections(C.Structure):
    _fields_ = [("A", _dp), ("Iy", _dp), ("Iz", _dp), ("J", _dp), ("t", _dp)]


class sso_materials(C.Structure):
    _fields_ = [("E", _dp), ("nu", _dp), ("G", _dp)]


class sso_supports(C.Structure):
    _fields_ = [("n", C.c_int32), ("node", _ip), ("mask6", _up)]


class sso_options(C.Structure):
    _fields_ = [("rtol", C.c_double), ("max_iter", C.c_int64), ("drill_alpha", C.c_double),
                ("warm_start", C.c_int32), ("check_every", C.c_int32), ("mem", C.c_int),
                ("cuda_stream", C.c_void_p), ("device", C.c_int32),
                ("n_parts", C.c_int32), ("part_ranges", _ip), ("nranks", C.c_int32),
                ("rank", C.c_int32), ("nccl_unique_id", C.c_void_p), ("batch", C.c_int32),
                ("reliable", C.c_int32), ("assembly", C.c_int32),
                ("storage", C.c_int32), ("precond", C.c_int32)]


class sso_solve_info(C.Structure):
    _fields_ = [("iters", C.c_int64), ("rel_res", C.c_double), ("true_rel_res", C.c_double),
                ("ms", C.c_double), ("status", C.c_int32), ("lanczos_iters", C.c_int32),
                ("lanczos_lmin", C.c_double), ("lanczos_lmax", C.c_double),
                ("err_energy_est", C.c_double), ("err2_est", C.c_double)]

    def as_dict(self):
        return dict(iters=self.iters, rel_res=self.rel_res, true_rel_res=self.true_rel_res,
                    ms=self.ms, status=self.status, lanczos_iters=self.lanczos_iters,
                    lanczos_lmin=self.lanczos_lmin, lanczos_lmax=self.lanczos_lmax,
                    err_energy_est=self.err_energy_est, err2_est=self.err2_est)


_H = C.c_void_p
_sig = {
    "sso_options_default": (C.c_int, [C.POINTER(sso_options)]),
    "sso_create": (C.c_int, [C.POINTER(sso_mesh), C.POINTER(sso_sections), C.POINTER(sso_materials),
                             C.POINTER(sso_supports), C.POINTER(sso_options), C.POINTER(_H)]),
    "sso_set_design": (C.c_int, [_H, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    "sso_set_stream": (C.c_int, [_H, C.c_void_p, C.c_int]),
    "sso_assemble": (C.c_int, [_H]),
    "sso_solve": (C.c_int, [_H, C.c_void_p, C.c_void_p, C.POINTER(sso_solve_info)]),
    "sso_grad": (C.c_int, [_H, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p]),
    "sso_grad_at": (C.c_int, [_H, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    "sso_spmv": (C.c_int, [_H, C.c_void_p, C.c_void_p]),
    "sso_grad_E": (C.c_int, [_H, C.c_int, C.c_void_p]),
    "sso_adjoint_solve": (C.c_int, [_H, C.c_void_p, C.c_void_p, C.POINTER(sso_solve_info)]),
    "sso_grad_adjoint": (C.c_int, [_H, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    "sso_set_material": (C.c_int, [_H, C.c_void_p]),
    "sso_set_density": (C.c_int, [_H, C.c_void_p, C.c_double, C.c_void_p, C.c_void_p]),
    "sso_grad_density": (C.c_int, [_H, C.c_int, C.c_void_p]),
    "sso_set_prescribed": (C.c_int, [_H, C.c_void_p]),
    "sso_set_area_load": (C.c_int, [_H, C.c_void_p, C.c_void_p, C.c_void_p]),
    "sso_hat_filter": (C.c_int, [_H, C.c_int32, C.c_double, C.c_int32, C.c_void_p, C.c_void_p]),
    "sso_sizes": (C.c_int, [_H, _lp, _lp, _lp]),
    "sso_export_csr": (C.c_int, [_H, C.c_void_p, C.c_void_p, C.c_void_p]),
    "sso_export_scatter": (C.c_int, [_H, C.c_void_p]),
    "sso_export_ke": (C.c_int, [_H, C.c_int64, C.c_int64, C.c_void_p]),
    "sso_export_dinv": (C.c_int, [_H, C.c_void_p]),
    "sso_profile_enable": (C.c_int, [_H, C.c_int32]),
    "sso_profile_read": (C.c_int, [_H, C.c_char_p, _dp, _lp]),
    "sso_profile_reset": (C.c_int, [_H]),
    "sso_launch_count": (C.c_int64, [_H]),
    "sso_part_info": (C.c_int, [_H, _ip, _ip, _ip, _ip]),
    "sso_storage_info": (C.c_int, [_H, _lp, _lp, _ip]),
    "sso_nccl_unique_id": (C.c_int, [C.c_void_p]),
    "sso_local_pattern": (C.c_int, [C.POINTER(sso_mesh), _ip, C.c_int32, C.c_int32, _lp, C.c_void_p, C.c_void_p]),
    "sso_halo_plan": (C.c_int, [C.POINTER(sso_mesh), _ip, C.c_int32, C.c_int32, _ip, C.c_void_p, _ip,
                                C.c_void_p, C.c_void_p, C.c_void_p]),
    "sso_last_error": (C.c_char_p, [_H]),
    "sso_destroy": (None, [_H]),
}
EXPORTED = tuple(_sig)
for _name, (_res, _args) in _sig.items():
    _fn = getattr(_lib, _name)
    _fn.restype = _res
    _fn.argtypes = _args


class SSOError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"{STATUS_NAMES.get(code, code)}: {msg}")
        self.code = code


_TORCH_DT = {np.dtype(np.float64): "torch.float64", np.dtype(np.int32): "torch.int32",
             np.dtype(np.uint8): "torch.uint8"}


def _ptr(a, dtype, n=None, device=None):
    """Pointer of a numpy array or torch tensor after checking what the C ABI relies on:
    dtype, C-contiguity, at least n elements and (tensors) the handle's device.  Raises
    ValueError instead of letting the library read or write out of bounds."""
    if a is None:
        return None
    dtype = np.dtype(dtype)
    if isinstance(a, np.ndarray):
        if a.dtype != dtype or not a.flags["C_CONTIGUOUS"]:
            raise ValueError(f"expected a C-contiguous {dtype} array, got {a.dtype} "
                             f"(contiguous={a.flags['C_CONTIGUOUS']})")
        if n is not None and a.size < n:
            raise ValueError(f"array has {a.size} elements, the call needs {n}")
        return a.ctypes.data
    if not hasattr(a, "data_ptr"):
        raise ValueError(f"expected a numpy array or torch tensor, got {type(a).__name__}")
    if str(a.dtype) != _TORCH_DT[dtype]:
        raise ValueError(f"expected a {_TORCH_DT[dtype]} tensor, got {a.dtype}")
    if not a.is_contiguous():
        raise ValueError("tensor must be contiguous")
    if n is not None and a.numel() < n:
        raise ValueError(f"tensor has {a.numel()} elements, the call needs {n}")
    if a.is_cuda and device is not None and a.device.index != device:
        raise ValueError(f"tensor on cuda:{a.device.index}, the handle lives on cuda:{device}")
    if not a.is_cuda:
        # a CPU tensor is host memory: only valid in host mode (checked by _mode)
        pass
    return a.data_ptr()


def _np(a, dtype):
    if a is None:
        return None
    return np.ascontiguousarray(a, dtype=dtype)


def _is_device(a):
    return a is not None and not isinstance(a, np.ndarray) and getattr(a, "is_cuda", False)


class Model:
    """One sso_handle.  `problem` is a dict as produced by workloads.* (x, y, z,
    beam_conn, quad_conn, A, Iy, Iz, J, t, E, nu, G, sup_node, sup_mask)."""

    def __init__(self, problem, rtol=1e-10, max_iter=200000, drill_alpha=1e-3, check_every=64,
                 warm_start=False, stream=None, device=-1, n_parts=1, part_ranges=None,
                 nranks=1, rank=0, nccl_id=None, batch=1, reliable=1, assembly=0, storage=0,
                 precond=0):
        P = problem
        self._keep = []
        x, y, z = (_np(P[k], np.float64) for k in ("x", "y", "z"))
        bc = _np(P["beam_conn"], np.int32).reshape(-1)
        qc = _np(P["quad_conn"], np.int32).reshape(-1)
        nb, nq = len(bc) // 2, len(qc) // 4
        A, Iy, Iz, J, t = (_np(P.get(k), np.float64) for k in ("A", "Iy", "Iz", "J", "t"))
        E, nu = _np(P["E"], np.float64), _np(P["nu"], np.float64)
        G = _np(P.get("G"), np.float64)
        sn, sm = _np(P["sup_node"], np.int32), _np(P["sup_mask"], np.uint8)
        self._keep += [x, y, z, bc, qc, A, Iy, Iz, J, t, E, nu, G, sn, sm]

        def dp(a):
            return None if a is None or a.size == 0 else a.ctypes.data_as(_dp)

        def ip(a):
            return None if a is None or a.size == 0 else a.ctypes.data_as(_ip)

        mesh = sso_mesh(len(x), dp(x), dp(y), dp(z), nb, ip(bc), nq, ip(qc))
        sec = sso_sections(dp(A), dp(Iy), dp(Iz), dp(J), dp(t))
        mat = sso_materials(dp(E), dp(nu), dp(G))
        sup = sso_supports(len(sn), ip(sn), sm.ctypes.data_as(_up) if sm.size else None)
        opt = sso_options()
        _lib.sso_options_default(C.byref(opt))
        opt.rtol, opt.max_iter, opt.drill_alpha = rtol, max_iter, drill_alpha
        opt.check_every, opt.warm_start, opt.device = check_every, int(warm_start), device
        opt.mem = MEM_HOST
        opt.cuda_stream = stream
        opt.n_parts, opt.nranks, opt.rank, opt.batch = n_parts, nranks, rank, batch
        opt.reliable, opt.assembly, opt.storage = reliable, assembly, storage
        opt.precond = precond
        if part_ranges is not None:
            pr = np.ascontiguousarray(part_ranges, np.int32)
            self._keep.append(pr)
            opt.part_ranges = pr.ctypes.data_as(_ip)
        if nccl_id is not None:
            idb = C.create_string_buffer(bytes(nccl_id), 128)
            self._keep.append(idb)
            opt.nccl_unique_id = C.cast(idb, C.c_void_p)
        h = _H()
        rc = _lib.sso_create(C.byref(mesh), C.byref(sec), C.byref(mat), C.byref(sup), C.byref(opt),
                             C.byref(h))
        if rc != SSO_OK:
            raise SSOError(rc, _lib.sso_last_error(None).decode())
        self.h = h
        self.g_nodes, self.g_quads = len(x), nq
        a, b, c, d = C.c_int32(), C.c_int32(), C.c_int32(), C.c_int32()
        _lib.sso_part_info(h, C.byref(a), C.byref(b), C.byref(c), C.byref(d))
        self.n_parts_here, self.own_node_begin = a.value, b.value
        # extents of this handle's f / u / gradient buffers (global unless multi-rank)
        self.n_nodes, self.n_beams, self.n_quads = c.value, nb, d.value
        self.ndof = 6 * c.value
        self.batch = batch
        self._mem = MEM_HOST
        self._stream = stream
        self._dev_opt = device
        self._device_idx = device if device >= 0 else None
        if self._device_idx is None:  # the device sso_create made current (-1: the caller's current)
            try:
                import torch
                self._device_idx = torch.cuda.current_device()
            except Exception:
                self._device_idx = None

    # -- plumbing ----------------------------------------------------------
    def _check(self, rc):
        if rc != SSO_OK:
            raise SSOError(rc, _lib.sso_last_error(self.h).decode())
        return rc

    def _mode(self, *arrays):
        """Pointer kind of this call's buffers: all device (torch CUDA tensors) or all host.
        Device mode orders the library after torch's current stream: a side stream is handed
        over as the handle's stream; torch's default (legacy) stream is passed as NULL, which
        makes every entry point wait for the work queued on it and it for the library's
        (include/sso.h sso_set_stream)."""
        given = [a for a in arrays if a is not None]
        devs = [_is_device(a) for a in given]
        if any(devs) and not all(devs):
            raise ValueError("mixed host and device buffers in one call")
        dev = bool(devs) and all(devs)
        mem = MEM_DEVICE if dev else MEM_HOST
        stream = None
        if dev:
            import torch
            want = self._device_index()
            for a in given:
                if a.device.index != want:
                    raise ValueError(f"tensor on cuda:{a.device.index}, the handle lives on cuda:{want}")
            stream = torch.cuda.current_stream(want).cuda_stream or None
        if mem != self._mem or (dev and stream != self._stream) or (dev and stream is None):
            self._check(_lib.sso_set_stream(self.h, stream, mem))
            self._mem, self._stream = mem, (stream if dev else self._stream)
        return dev

    def _device_index(self):
        if self._device_idx is None:
            import torch
            self._device_idx = self._dev_opt if self._dev_opt >= 0 else torch.cuda.current_device()
        return self._device_idx

    def close(self):
        if getattr(self, "h", None):
            _lib.sso_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- ABI -----------------------------------------------------------------
    def sizes(self):
        a, b, c = C.c_int64(), C.c_int64(), C.c_int64()
        self._check(_lib.sso_sizes(self.h, C.byref(a), C.byref(b), C.byref(c)))
        return a.value, b.value, c.value

    def storage_info(self):
        v, b, s = C.c_int64(), C.c_int64(), C.c_int32()
        self._check(_lib.sso_storage_info(self.h, C.byref(v), C.byref(b), C.byref(s)))
        return v.value, b.value, s.value  # 0 full, 2 two-pass symmetric, 3 pull symmetric

    def set_design(self, x=None, y=None, z=None, t=None):
        dev = self._mode(x, y, z, t)
        conv = (lambda a: a) if dev else (lambda a: _np(a, np.float64))
        arrs = [None if a is None else conv(a) for a in (x, y, z, t)]
        ns = [self.batch * self.g_nodes] * 3 + [self.batch * self.g_quads]
        self._check(_lib.sso_set_design(self.h, *[_ptr(a, np.float64, n) for a, n in zip(arrs, ns)]))

    def assemble(self):
        self._check(_lib.sso_assemble(self.h))

    def solve(self, f, u=None, raise_on_error=True):
        """Returns (u, info dict) — with batch > 1, u is [B, ndof] and info a list of B dicts.
        f, u: numpy (host) or torch CUDA tensors (device)."""
        dev = self._mode(f, u)
        shape = (self.batch, self.ndof) if self.batch > 1 else (self.ndof,)
        if not dev:
            f = _np(f, np.float64)
            if u is None:
                u = np.zeros(shape)
        elif u is None:
            import torch
            u = torch.zeros(shape, dtype=torch.float64, device=f.device)
        infos = (sso_solve_info * self.batch)()
        nv = self.batch * self.ndof
        rc = _lib.sso_solve(self.h, _ptr(f, np.float64, nv), _ptr(u, np.float64, nv), infos)
        if raise_on_error:
            self._check(rc)
        if self.batch > 1:
            return u, [i.as_dict() for i in infos]
        return u, infos[0].as_dict()

    def grad(self, objective=OBJ_COMPLIANCE, out=None):
        """Returns (C, dC_dxyz [3, n_nodes], dC_dt [n_quads]) for the last solve."""
        return self._grad(objective, None, None, out)

    def grad_at(self, f, u, objective=OBJ_COMPLIANCE, out=None):
        return self._grad(objective, f, u, out)

    def _grad(self, objective, f, u, out):
        dev = self._mode(f, u, *(out or ()))
        B = self.batch
        if out is None:
            if dev:
                import torch
                ref = f if f is not None else u
                Cv = torch.zeros(B, dtype=torch.float64, device=ref.device)
                dX = torch.zeros(B * 3 * self.n_nodes, dtype=torch.float64, device=ref.device)
                dT = torch.zeros(B * max(self.n_quads, 1), dtype=torch.float64, device=ref.device)
            else:
                Cv, dX, dT = np.zeros(B), np.zeros(B * 3 * self.n_nodes), np.zeros(B * max(self.n_quads, 1))
        else:
            Cv, dX, dT = out
        nX, nT = B * 3 * self.n_nodes, B * self.n_quads
        if f is None:
            rc = _lib.sso_grad(self.h, objective, _ptr(Cv, np.float64, B), _ptr(dX, np.float64, nX),
                               _ptr(dT, np.float64, nT))
        else:
            if not dev:
                f, u = _np(f, np.float64), _np(u, np.float64)
            nv = B * self.ndof
            rc = _lib.sso_grad_at(self.h, objective, _ptr(f, np.float64, nv), _ptr(u, np.float64, nv),
                                  _ptr(Cv, np.float64, B), _ptr(dX, np.float64, nX), _ptr(dT, np.float64, nT))
        self._check(rc)
        if out is not None:
            return out
        if B > 1:
            return Cv, dX.reshape(B, 3, self.n_nodes), dT.reshape(B, -1)[:, : self.n_quads]
        C0 = float(Cv[0]) if not dev else Cv
        return C0, dX.reshape(3, self.n_nodes), dT[: self.n_quads]

    def grad_E(self, objective=OBJ_COMPLIANCE):
        """dC/dE per element (beams first, then quads), [batch, n_elems] or [n_elems]."""
        ne = self.n_beams + self.g_quads
        out = np.zeros(self.batch * ne)
        self._mode()
        self._check(_lib.sso_grad_E(self.h, objective, out.ctypes.data))
        return out.reshape(self.batch, ne) if self.batch > 1 else out

    def adjoint_solve(self, dg_du):
        """lambda with K lambda = dg/du (primal state kept).  Returns (lambda, info); with
        batch > 1, dg_du and lambda are [B, ndof] and info a list of B dicts."""
        self._mode()
        B = self.batch
        g = _np(dg_du, np.float64)
        lam = np.zeros(B * self.ndof)
        infos = (sso_solve_info * B)()
        self._check(_lib.sso_adjoint_solve(self.h, g.ctypes.data, lam.ctypes.data, infos))
        if B > 1:
            return lam.reshape(B, self.ndof), [i.as_dict() for i in infos]
        return lam, infos[0].as_dict()

    def grad_adjoint(self, lam):
        """(-lambda^T dK/dX u [3, n], -lambda^T dK/dt u [n_quads], -lambda^T dK/dE u [n_elems]);
        with batch > 1 each gets a leading design axis."""
        self._mode()
        B = self.batch
        lam = _np(lam, np.float64)
        ne = self.n_beams + self.g_quads
        dX = np.zeros(B * 3 * self.n_nodes)
        dT = np.zeros(B * max(self.n_quads, 1))
        dE = np.zeros(B * ne)
        self._check(_lib.sso_grad_adjoint(self.h, lam.ctypes.data, dX.ctypes.data, dT.ctypes.data,
                                          dE.ctypes.data))
        if B > 1:
            return dX.reshape(B, 3, self.n_nodes), dT.reshape(B, -1)[:, : self.n_quads], dE.reshape(B, ne)
        return dX.reshape(3, self.n_nodes), dT[: self.n_quads], dE

    def set_density(self, rho, penal, E0, G0=None):
        """SIMP densities (Eq. 12): E = rho^P E0 (G = rho^P G0, or derived from nu),
        per element, beams first.  Requires a new assemble()."""
        dev = self._mode(rho)
        if not dev:
            rho, E0 = _np(rho, np.float64), _np(E0, np.float64)
            G0 = None if G0 is None else _np(G0, np.float64)
        self._check(_lib.sso_set_density(self.h, _ptr(rho, np.float64), float(penal), _ptr(E0, np.float64),
                                         None if G0 is None else _ptr(G0, np.float64)))

    def grad_density(self, objective=OBJ_COMPLIANCE):
        """dC/drho per element (beams first, then quads) after set_density, [batch, n_elems]
        or [n_elems]."""
        ne = self.n_beams + self.g_quads
        out = np.zeros(self.batch * ne)
        self._mode()
        self._check(_lib.sso_grad_density(self.h, objective, out.ctypes.data))
        return out.reshape(self.batch, ne) if self.batch > 1 else out

    def set_material(self, E):
        dev = self._mode(E)
        if not dev:
            E = _np(E, np.float64)
        self._check(_lib.sso_set_material(self.h, _ptr(E, np.float64)))

    def set_prescribed(self, b):
        """Prescribed support displacements b [6 n_nodes] ([B, 6 n_nodes] for a batch;
        constrained entries used); None switches them off.  Requires a new assemble()."""
        dev = self._mode(b)
        if b is not None and not dev:
            b = _np(b, np.float64)
        self._check(_lib.sso_set_prescribed(self.h, _ptr(b, np.float64)))

    def set_area_load(self, q=None, w=None, direction=(0.0, 0.0, -1.0)):
        """Design-dependent area load (include/sso.h sso_set_area_load): per-quad load per
        unit area q and unit weight w (self-weight w t) along `direction`; q = w = None
        switches it off."""
        dev = self._mode(q, w)
        if not dev:
            q, w = _np(q, np.float64), _np(w, np.float64)
        d = np.ascontiguousarray(direction, dtype=np.float64)
        assert d.shape == (3,)
        self._check(_lib.sso_set_area_load(self.h, _ptr(q, np.float64), _ptr(w, np.float64), d.ctypes.data))

    def hat_filter(self, values, radius, on_elements=False):
        """Hat filter of sensitivities (include/sso.h sso_hat_filter): values [n] or
        [ncomp<=3, n] over nodes (n_nodes) or element centroids (n_beams + n_quads); with
        batch > 1 a leading design axis ([B, n] or [B, ncomp, n]), each design filtered over
        its own coordinates."""
        dev = self._mode(values)
        if dev:
            import torch
            v = values.contiguous()
            out = torch.empty_like(v)
        else:
            v = _np(values, np.float64)
            out = np.empty_like(v)
        lead = 1 if self.batch > 1 else 0
        ncomp = 1 if v.ndim == 1 + lead else int(v.shape[lead])
        self._check(_lib.sso_hat_filter(self.h, 1 if on_elements else 0, float(radius), ncomp,
                                        _ptr(v, np.float64), _ptr(out, np.float64)))
        return out

    def spmv(self, x):
        dev = self._mode(x)
        if dev:
            import torch
            y = torch.empty_like(x)
        else:
            x = _np(x, np.float64)
            y = np.empty_like(x)
        nv = self.batch * self.ndof
        self._check(_lib.sso_spmv(self.h, _ptr(x, np.float64, nv), _ptr(y, np.float64, nv)))
        return y

    def export_csr(self, values=True):
        ndof, nnz, _ = self.sizes()
        rp = np.empty(ndof + 1, np.int64)
        ci = np.empty(nnz, np.int32)
        v = np.empty(nnz, np.float64) if values else None
        self._check(_lib.sso_export_csr(self.h, rp.ctypes.data, ci.ctypes.data,
                                        None if v is None else v.ctypes.data))
        return rp, ci, v

    def export_scatter(self):
        br = np.empty(4 * self.n_beams + 16 * self.n_quads, np.int32)
        self._check(_lib.sso_export_scatter(self.h, br.ctypes.data))
        return br

    def export_ke(self, first, count):
        if first < self.n_beams:
            assert first + count <= self.n_beams, "export beams and quads separately"
            m = 12
        else:
            m = 24
        ke = np.empty((count, m, m))
        self._check(_lib.sso_export_ke(self.h, first, count, ke.ctypes.data))
        return ke

    def export_dinv(self):
        d = np.empty(self.ndof)
        self._check(_lib.sso_export_dinv(self.h, d.ctypes.data))
        return d

    def profile_enable(self, on=True):
        self._check(_lib.sso_profile_enable(self.h, int(on)))

    def profile_reset(self):
        self._check(_lib.sso_profile_reset(self.h))

    def profile_read(self, name):
        ms, n = C.c_double(), C.c_int64()
        self._check(_lib.sso_profile_read(self.h, name.encode(), C.byref(ms), C.byref(n)))
        return ms.value, n.value

    def launch_count(self):
        return int(_lib.sso_launch_count(self.h))


def last_create_error():
    return _lib.sso_last_error(None).decode()


def nccl_unique_id():
    buf = C.create_string_buffer(128)
    rc = _lib.sso_nccl_unique_id(buf)
    if rc != SSO_OK:
        raise SSOError(rc, last_create_error())
    return buf.raw


def _mesh_struct(P):
    x, y, z = (np.ascontiguousarray(P[k], np.float64) for k in ("x", "y", "z"))
    bc = np.ascontiguousarray(P["beam_conn"], np.int32).reshape(-1)
    qc = np.ascontiguousarray(P["quad_conn"], np.int32).reshape(-1)
    keep = [x, y, z, bc, qc]
    m = sso_mesh(len(x), x.ctypes.data_as(_dp), y.ctypes.data_as(_dp), z.ctypes.data_as(_dp),
                 len(bc) // 2, bc.ctypes.data_as(_ip) if bc.size else None,
                 len(qc) // 4, qc.ctypes.data_as(_ip) if qc.size else None)
    return m, keep


def local_pattern(P, ranges, part):
    """Host-only: CSR pattern (row_ptr, col_idx in global ids) of strip `part`'s owned rows."""
    m, keep = _mesh_struct(P)
    rg = np.ascontiguousarray(ranges, np.int32)
    n_parts = len(rg) - 1
    nnz = C.c_int64()
    rc = _lib.sso_local_pattern(C.byref(m), rg.ctypes.data_as(_ip), n_parts, part, C.byref(nnz), None, None)
    if rc != SSO_OK:
        raise SSOError(rc, last_create_error())
    n_own = int(rg[part + 1] - rg[part])
    rp = np.empty(6 * n_own + 1, np.int64)
    ci = np.empty(nnz.value, np.int32)
    rc = _lib.sso_local_pattern(C.byref(m), rg.ctypes.data_as(_ip), n_parts, part, C.byref(nnz),
                                rp.ctypes.data, ci.ctypes.data)
    if rc != SSO_OK:
        raise SSOError(rc, last_create_error())
    return rp, ci


def halo_plan(P, ranges, part):
    """Host-only: (halo_gid, {neighbour: send_gid array}) of strip `part`."""
    m, keep = _mesh_struct(P)
    rg = np.ascontiguousarray(ranges, np.int32)
    n_parts = len(rg) - 1
    nh, nn = C.c_int32(), C.c_int32()
    rc = _lib.sso_halo_plan(C.byref(m), rg.ctypes.data_as(_ip), n_parts, part, C.byref(nh), None,
                            C.byref(nn), None, None, None)
    if rc != SSO_OK:
        raise SSOError(rc, last_create_error())
    halo = np.empty(nh.value, np.int32)
    nbr = np.empty(nn.value, np.int32)
    cnt = np.empty(nn.value, np.int32)
    rc = _lib.sso_halo_plan(C.byref(m), rg.ctypes.data_as(_ip), n_parts, part, C.byref(nh),
                            halo.ctypes.data, C.byref(nn), nbr.ctypes.data, cnt.ctypes.data, None)
    send = np.empty(int(cnt.sum()), np.int32)
    rc = _lib.sso_halo_plan(C.byref(m), rg.ctypes.data_as(_ip), n_parts, part, C.byref(nh),
                            halo.ctypes.data, C.byref(nn), nbr.ctypes.data, cnt.ctypes.data,
                            send.ctypes.data)
    out, off = {}, 0
    for k in range(nn.value):
        out[int(nbr[k])] = send[off:off + cnt[k]].copy()
        off += cnt[k]
    return halo, out
