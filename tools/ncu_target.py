"""Short ncu target: C3b assemble + 128 CG iterations (direct launches) + gradient.
SSO_STORAGE selects sso_options.storage (default 0 = library default)."""
import os
import sys
sys.path.insert(0, '.')
import workloads as W
import paper_2407_20026_b200 as sso
P = W.config3b()
m = sso.Model(P, rtol=1e-10, max_iter=128, check_every=64, storage=int(os.environ.get("SSO_STORAGE", "0")))
m.assemble()
m.profile_enable(True)   # direct (non-graph) launches so every kernel is visible
u, info = m.solve(P["f"], raise_on_error=False)
C, dX, dT = m.grad_at(P["f"], u)
print("ok", info["iters"])
