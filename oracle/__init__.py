"""CPU fp64 ORACLE for the JAX-SSO hot path (arXiv 2407.20026).

TEST INFRASTRUCTURE ONLY.  Only `tests/`, `__graft_entry__.smoke()` and the
`cpu_baseline` / `--impl reference` legs of `bench.py` may import, call or
execute anything in this package.  The product path
(`paper_2407_20026_b200/`) never imports it and has no CPU fallback.

The oracle is plain, slow and written to be checked against the paper by eye:
explicit loops over elements, nodes and Gauss points; a dict-of-keys global
matrix; dense Cholesky (small) or textbook Jacobi-PCG (large); exact
derivatives of element matrices by complex step.  It shares no code, header,
table or constant generator with the CUDA path; the only module both sides
use is `workloads/`, which generates seeded inputs and holds none of the
method's arithmetic.

Modules (each function cites the passage it follows):
    beam      3D Euler-Bernoulli frame element (reading C1)
    shell     flat 4-node MITC-4 shell element (reading C2)
    assembly  DOK assembly, CSR pattern, scatter map, supports
    solve     dense Cholesky, Lagrange-multiplier LU, Jacobi-PCG
    grad      compliance and adjoint gradient
    filter    hat filter of sensitivities (reading c16)
    loads     design-dependent area loads, 2 u^T df/dp term (reading c17)
    prescribed  non-zero support displacements V u = b via the Lagrange system (reading c18)

Pins (tests/test_oracle_*.py, run with -m "not gpu") tie every function to
something other than itself: closed-form cantilever results, the Navier plate
series, patch tests, exact rigid-body null spaces, brute-force pattern sets,
Lagrange-vs-elimination equivalence, global complex-step and central finite
differences, homogeneity identities and the paper's barrel-arch numbers.
Functions without such a pin say "parity unpinned" in their docstring.
"""
from . import beam, shell, assembly, solve, grad, filter, loads, prescribed  # noqa: F401
