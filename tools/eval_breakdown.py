"""Wall-clock breakdown of one C3b evaluation (assemble / solve / grad), device-resident
inputs, synchronised around each phase; solve's info["ms"] is the CG loop's device time."""
import sys, time, json
sys.path.insert(0, '.')
import numpy as np, torch
import workloads as W
import paper_2407_20026_b200 as sso
P = W.config3b()
m = sso.Model(P, rtol=1e-10, device=0)
f = torch.from_numpy(P["f"]).cuda()
u = torch.zeros_like(f)
C = torch.zeros(1, dtype=torch.float64, device="cuda")
dX = torch.zeros(3 * m.n_nodes, dtype=torch.float64, device="cuda")
dT = torch.zeros(m.n_quads, dtype=torch.float64, device="cuda")
for rep in range(3):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    m.assemble(); torch.cuda.synchronize(); t1 = time.perf_counter()
    _, info = m.solve(f, u); torch.cuda.synchronize(); t2 = time.perf_counter()
    m.grad(0, out=(C, dX, dT)); torch.cuda.synchronize(); t3 = time.perf_counter()
    print(json.dumps({"assemble_ms": 1e3 * (t1 - t0), "solve_ms": 1e3 * (t2 - t1), "cg_device_ms": info["ms"],
                      "iters": info["iters"], "grad_ms": 1e3 * (t3 - t2), "total_ms": 1e3 * (t3 - t0),
                      "us_per_iter_device": 1e3 * info["ms"] / info["iters"]}))
