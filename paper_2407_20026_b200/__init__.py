"""B200-native hot path of JAX-SSO (arXiv 2407.20026): batched fp64 element
stiffness (3D frame + MITC-4 shell), atomic-free CSR assembly with supports,
Jacobi-PCG, and the element-wise adjoint gradient of compliance — all as
hand-written sm_100a CUDA kernels behind the C ABI in include/sso.h.

This package holds the CUDA sources (csrc/), the nvcc build (build.py) and the
ctypes binding (api.py).  It never imports `oracle/` and has no CPU fallback.
"""
from .api import (Model, SSOError, OBJ_COMPLIANCE, OBJ_STRAIN_ENERGY, MEM_HOST, MEM_DEVICE,  # noqa: F401
                  LIB_PATH, EXPORTED, last_create_error, nccl_unique_id, local_pattern,
                  halo_plan)
