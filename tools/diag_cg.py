"""Diagnostic: CG iteration counts / residual gap vs rtol on the shell family (GPU)."""
import sys, time, json
import numpy as np
import torch
sys.path.insert(0, '.')
import workloads as W
import paper_2407_20026_b200 as sso

def run(P, rtols, dev):
    out = []
    m = sso.Model(P, rtol=rtols[0])
    m.assemble()
    for rt in rtols:
        m2 = sso.Model(P, rtol=rt)
        m2.assemble()
        f = torch.from_numpy(P["f"]).cuda() if dev else P["f"]
        t0 = time.perf_counter()
        u, info = m2.solve(f, raise_on_error=False)
        torch.cuda.synchronize()
        info["wall_s"] = time.perf_counter() - t0
        info["rtol"] = rt
        out.append(info)
        print(P["name"], json.dumps(info), flush=True)
        m2.close()
    return out

if __name__ == "__main__":
    for n in (50, 100, 200, 408):
        P = W.shell_config3(n, cfg=3)
        run(P, [1e-8, 1e-10, 1e-12], dev=(n == 100))
