"""Per-iteration cost of the strips' NCCL algorithm on ONE GPU (1-rank communicator,
SSO_NCCL_SELF=1) against the single-part solve: python tools/nccl_self_time.py [N] [SUP]"""
import os
import sys
sys.path.insert(0, '.')
import torch
import workloads as W
import paper_2407_20026_b200 as sso
n = int(sys.argv[1]) if len(sys.argv) > 1 else 408
sup = sys.argv[2] if len(sys.argv) > 2 else "clamped_edges"
P = W.shell_config3(n, cfg=4 if sup == "c4" else 3, supports=sup)
f = torch.from_numpy(P["f"]).cuda()
for mode in ("local", "nccl-1rank"):
    kw = {}
    if mode != "local":
        os.environ["SSO_NCCL_SELF"] = "1"
        kw = dict(nranks=1, rank=0, nccl_id=sso.nccl_unique_id())
    m = sso.Model(P, rtol=1e-10, max_iter=int(os.environ.get("MAXIT", "3000")), **kw)
    os.environ.pop("SSO_NCCL_SELF", None)
    m.assemble()
    u = torch.zeros_like(f)
    m.solve(f, u, raise_on_error=False)
    ts = []
    for _ in range(2):
        _, info = m.solve(f, u, raise_on_error=False)
        ts.append(info["ms"])
    print(f"{mode:12s} n={n}: {info['iters']} iterations, {1000 * min(ts) / info['iters']:.1f} us/iter", flush=True)
    m.close()
