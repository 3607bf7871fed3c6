"""Solve-only timing at C3b: iterations, ms per solve, sampled SpMV launch time."""
import json, os, sys
sys.path.insert(0, '.')
import numpy as np
import torch
import workloads as W
import paper_2407_20026_b200 as sso
n = int(os.environ.get("N", "408"))
sup = os.environ.get("SUP", "clamped_edges")
P = W.shell_config3(n, cfg=4 if sup == "c4" else 3, supports=sup)
m = sso.Model(P, rtol=1e-10, n_parts=int(os.environ.get("PARTS", "1")),
              reliable=int(os.environ.get("REL", "1")), storage=int(os.environ.get("STORAGE", "0")),
              precond=int(os.environ.get("PRECOND", "0")), max_iter=int(os.environ.get("MAXIT", "200000")))
m.assemble()
f = torch.from_numpy(P["f"]).cuda()
u = torch.zeros_like(f)
m.solve(f, u, raise_on_error=False)
m.profile_enable(True)
m.profile_reset()
ts = []
for _ in range(int(os.environ.get("REPS", "3"))):
    _, info = m.solve(f, u, raise_on_error=False)
    ts.append(info["ms"])
ms, cnt = m.profile_read("spmv")
ndof, nnz, nb = m.sizes()
sv, sb, kind = m.storage_info()
byts = 8 * sv + 4 * sb + 8 * (m.n_nodes + 1) + 16 * ndof if kind != 3 else 8 * sv + 4 * sb + 64 * m.n_nodes + 16 * ndof
avg = ms / max(cnt, 1)
print(json.dumps({"precond": os.environ.get("PRECOND", "0"), "variant": os.environ.get("SSO_SPMV_VARIANT", "0"), "rel": os.environ.get("REL", "1"), "storage": os.environ.get("STORAGE", "0"),
                  "sup": sup, "n": n, "parts": os.environ.get("PARTS", "1"), "coop": os.environ.get("SSO_COOP", "1"), "iters": info["iters"],
                  "solve_ms": min(ts), "us_per_iter": 1000 * min(ts) / (info["iters"] or int(os.environ.get("MAXIT", "1"))),
                  "spmv_us": 1000 * avg, "spmv_GBs": byts / (avg / 1000) / 1e9 if avg else 0,
                  "true_rel_res": info["true_rel_res"]}))
