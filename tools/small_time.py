"""Solve-only latency of the small configurations (C1, C2): python tools/small_time.py"""
import os
import sys
sys.path.insert(0, '.')
import workloads as W
import paper_2407_20026_b200 as sso
for name in ("config1", "config2"):
    P = getattr(W, name)()
    for ce in (64, 256):
        m = sso.Model(P, rtol=1e-10, check_every=ce)
        m.assemble()
        for _ in range(3):
            u, info = m.solve(P["f"])
        ts = []
        for _ in range(10):
            u, info = m.solve(P["f"])
            ts.append(info["ms"])
        t = min(ts)
        print(f"{name} check_every {ce}: {info['iters']} iterations, solve {t:.3f} ms, {1000 * t / info['iters']:.2f} us/iter, "
              f"SSO_SMALL={os.environ.get('SSO_SMALL', '1')}")
        m.close()
