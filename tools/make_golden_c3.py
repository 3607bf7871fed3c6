"""Write tests/golden/c3_oracle.npz: the CPU fp64 oracle's result on config C3 (200 x 200
MITC-4 quads, 242 406 DOF; BASELINE.json configs[2]).  With `c4` it
writes tests/golden/c4r120_oracle.npz instead: the C4 recipe (edge y = 0 clamped, two
pinned corners; BASELINE.json configs[3]) at n = 120 (87 846 DOF), whose conditioning is
the C4 one (one clamped edge instead of four).

Calls only oracle/ (and the seeded input generator workloads/): DOK assembly, supports by
elimination, the oracle's textbook Jacobi-PCG to rtol 1e-13 (SURVEY §8(c) C5 "CG for
large ones"), C = f^T u (C6), and the adjoint gradient (C7, complex-step dK_e/dp) at a
seeded sample of nodes and elements.  Stored: u (all 242 406 entries), C, the sampled
gradient components, and the oracle's iteration count / true residual as metadata.

    python tools/make_golden_c3.py        # ~5-10 min of CPU
    python tools/make_golden_c3.py c4     # the C4-recipe file
"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import workloads as W  # noqa: E402
from oracle import assembly as A, grad as G, solve as S  # noqa: E402

def main():
    c4 = len(sys.argv) > 1 and sys.argv[1] == "c4"
    OUT = os.path.join(ROOT, "tests", "golden", "c4r120_oracle.npz" if c4 else "c3_oracle.npz")
    t0 = time.time()
    P = W.shell_config3(120, cfg=4, supports="c4") if c4 else W.config3()
    nn, nq = len(P["x"]), len(P["quad_conn"])
    nd = 6 * nn
    dok = A.assemble_dok(P)
    row_ptr, col_idx, vals = A.csr_from_dok(dok, nd)
    del dok
    fixed = A.fixed_dofs(P)
    vals = A.apply_supports_csr(row_ptr, col_idx, vals, fixed)
    import scipy.sparse as sp
    K = sp.csr_matrix((vals, col_idx, row_ptr), shape=(nd, nd))
    fbc = P["f"].copy()
    fbc[fixed] = 0.0
    t1 = time.time()
    print(f"assembled {nq} quads, nnz {K.nnz} in {t1 - t0:.1f} s", flush=True)
    u, info = S.pcg(K, fbc, 1.0 / K.diagonal(), rtol=1e-13, max_iter=200000)
    t2 = time.time()
    print(f"PCG: {info['iters']} iterations, true rel res {info['true_rel_res']:.3e} in {t2 - t1:.1f} s",
          flush=True)
    C = G.compliance(P["f"], u)
    # seeded sample: 64 free interior nodes x 3 axes, 32 elements
    rng = np.random.default_rng(20240726)
    free_nodes = np.array([n for n in range(nn) if not fixed[6 * n]])
    nodes = np.sort(rng.choice(free_nodes, 64, replace=False))
    elems = np.sort(rng.choice(nq, 32, replace=False))
    X = A.coords(P)
    gX = np.zeros((len(nodes), 3))
    for k, n in enumerate(nodes):
        for e in A.incident_elements(P, int(n)):  # ascending element order
            part, _ = G.element_grad(P, e, u, 1.0, X)
            il = list(A.element_nodes(P, e)).index(n)
            gX[k] += part[il]
    gT = np.array([G.element_grad(P, int(e), u, 1.0, X)[1] for e in elems])
    t3 = time.time()
    print(f"gradient sample in {t3 - t2:.1f} s; C = {C:.12e}", flush=True)
    np.savez_compressed(OUT, u=u, C=np.array(C), grad_nodes=nodes, grad_X=gX, grad_elems=elems, grad_t=gT,
                        iters=np.array(info["iters"]), true_rel_res=np.array(info["true_rel_res"]),
                        rtol=np.array(1e-13))
    print(f"wrote {OUT} ({os.path.getsize(OUT) / 1e6:.1f} MB) in {time.time() - t0:.0f} s")


if __name__ == "__main__":
    main()
