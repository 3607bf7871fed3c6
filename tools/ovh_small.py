"""Fixed per-solve costs of a latency configuration (C1): solve time against the iteration
count, assembly and gradient times.  python tools/ovh_small.py"""
import sys
import time
sys.path.insert(0, '.')
import torch
import workloads as W
import paper_2407_20026_b200 as sso
P = W.config1()
for mi in (1, 2, 64, 100000):
    m = sso.Model(P, rtol=1e-10, max_iter=mi, check_every=64)
    m.assemble()
    for _ in range(3):
        u, info = m.solve(P["f"], raise_on_error=False)
    ts = []
    for _ in range(10):
        t0 = time.perf_counter()
        u, info = m.solve(P["f"], raise_on_error=False)
        ts.append(time.perf_counter() - t0)
    line = f"max_iter {mi}: {info['iters']} iterations, info.ms {info['ms']:.3f}, wall {1000 * min(ts):.3f} ms"
    if info["status"] == 0:
        t0 = time.perf_counter()
        for _ in range(20):
            m.grad()
        line += f", grad {(time.perf_counter() - t0) / 20 * 1000:.3f} ms"
    t0 = time.perf_counter()
    for _ in range(20):
        m.assemble()
    torch.cuda.synchronize()
    print(line + f", assemble {(time.perf_counter() - t0) / 20 * 1000:.3f} ms")
    m.close()
