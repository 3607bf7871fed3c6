"""Small end-to-end run for compute-sanitizer (C1 beams and C2 shell: assemble, point and
node-block Jacobi solves, gradient, general adjoint; C2 in 3 strips; a 3-design batch)."""
import sys
sys.path.insert(0, '.')
import numpy as np
import workloads as W
import paper_2407_20026_b200 as sso
for make in (W.config1, W.config2):
    P = make()
    for pc in (0, 1):
        m = sso.Model(P, rtol=1e-10, precond=pc)
        m.assemble()
        u, info = m.solve(P["f"])
        C, dX, dT = m.grad()
        lam, _ = m.adjoint_solve(u)
        m.grad_adjoint(lam)
        assert info["status"] == 0
P = W.config2()
m = sso.Model(P, rtol=1e-10, n_parts=3)
m.assemble()
u, info = m.solve(P["f"])
m.grad()
designs = [W.config5_design(b, n=8) for b in range(3)]
mb = sso.Model(designs[0], rtol=1e-10, batch=3)
mb.set_design(z=np.stack([d["z"] for d in designs]), t=np.stack([d["t"] for d in designs]))
mb.assemble()
mb.solve(np.stack([d["f"] for d in designs]))
mb.grad()
print("sanitize target ok")
