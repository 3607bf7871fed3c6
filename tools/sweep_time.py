"""Time plain SpMVs at C3b (CUDA events around 20 launches)."""
import os, sys, json
sys.path.insert(0, '.')
import numpy as np, torch
import workloads as W
import paper_2407_20026_b200 as sso
P = W.config3b()
m = sso.Model(P, rtol=1e-10)
m.assemble()
x = torch.from_numpy(np.random.default_rng(0).standard_normal(m.ndof)).cuda()
y = torch.empty_like(x)
for _ in range(3):
    m.spmv(x)
torch.cuda.synchronize()
m.profile_enable(True)
m.profile_reset()
for _ in range(20):
    m.spmv(x)
torch.cuda.synchronize()
ms, n = m.profile_read("spmv")
print(json.dumps({"dbg": os.environ.get("SSO_SWEEP_DBG", "0"), "sweep": os.environ.get("SSO_SWEEP", "1"),
                  "kernel": m.spmv_info(), "us_per_spmv": 1000 * ms / max(n, 1), "n": n}))
