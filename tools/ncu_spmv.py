"""ncu target: a few plain SpMVs at C3b through the default kernel (SSO_SWEEP selects)."""
import sys
sys.path.insert(0, '.')
import numpy as np
import torch
import workloads as W
import paper_2407_20026_b200 as sso
P = W.config3b()
m = sso.Model(P, rtol=1e-10)
m.assemble()
x = torch.from_numpy(np.random.default_rng(0).standard_normal(m.ndof)).cuda()
for _ in range(4):
    y = m.spmv(x)
torch.cuda.synchronize()
print("ok", m.spmv_info())
