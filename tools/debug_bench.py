import sys, torch, numpy as np
sys.path.insert(0, '.')
import workloads as W
import paper_2407_20026_b200 as sso
torch.cuda.set_device(0)
st = torch.cuda.current_stream()
print("torch stream handle", st.cuda_stream, flush=True)
for name, P in (("C3b", W.config3b()),):
    for use_stream in (False, True):
        try:
            m = sso.Model(P, rtol=1e-10, stream=st.cuda_stream if use_stream else None, device=0)
            m.assemble()
            f = torch.from_numpy(P["f"]).cuda()
            u = torch.zeros_like(f)
            _, info = m.solve(f, u)
            C = torch.zeros(1, dtype=torch.float64, device="cuda")
            dX = torch.zeros(3 * m.n_nodes, dtype=torch.float64, device="cuda")
            dT = torch.zeros(m.n_quads, dtype=torch.float64, device="cuda")
            m.grad(0, out=(C, dX, dT))
            print(name, use_stream, "ok", info["iters"], float(C), flush=True)
            m.close()
        except Exception as e:
            print(name, use_stream, "FAIL", e, flush=True)
