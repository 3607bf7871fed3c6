"""Benchmark: shell FEA solve + adjoint gradient evaluations per second at 1M DOF
(BASELINE.json metric; workload C3b = 408 x 408 MITC-4 quads, 1 003 686 DOF,
reading c15), one step = one full pass of the hot path: A1+A2 element
stiffness + assembly (sso_assemble), A3 Jacobi-PCG to rtol (sso_solve), A4
compliance + adjoint gradient (sso_grad).  A0 (pattern) runs once at create.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]

N > 1 runs under torchrun (one rank per GPU): the same C3b evaluation split
into N contiguous node strips, one per GPU, with the halo of p and the CG
scalars exchanged through NCCL every iteration (strong scaling; DESIGN.md
"Multi-GPU").  --virtual-parts P runs that partitioned algorithm with P strips
on one GPU (in-process transport).
`--impl reference` times the CPU oracle (oracle/) on a bounded sample of the
same workload on the host cores, extrapolated to the same metric.
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "shell FEA solve+adjoint grad evals/sec at 1M DOF; CG SpMV HBM GB/s vs peak"
UNIT = "evals/s"
N_GRID = 408
RTOL = 1e-10


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as fh:
            d = json.load(fh)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def ncu_traffic(storage_kind):
    """dram bytes per SpMV launch of the kernel this storage kind runs, from the committed
    ncu --set full capture (profiles/spmv_traffic.json), if any."""
    p = os.path.join(ROOT, "profiles", "spmv_traffic.json")
    if os.path.exists(p):
        with open(p) as fh:
            e = json.load(fh).get("by_storage", {}).get(str(storage_kind))
        return e.get("dram_bytes_per_launch") if e else None
    return None


class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        self.lines = []
        if self.proc:
            self.proc.terminate()
            try:
                out, _ = self.proc.communicate(timeout=5)
            except Exception:
                self.proc.kill()
                out = ""
            self.lines = [l for l in out.splitlines() if l.strip()]

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for l in getattr(self, "lines", []):
            parts = [p.strip() for p in l.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx = max(mx, float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm)}


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


# ----------------------------------------------------------------------------
# CPU oracle baseline (bounded sample, extrapolated to the C3b workload)
# ----------------------------------------------------------------------------

def oracle_sample(P, n_elem=2000, n_grad=1000, pcg_grid=60, pcg_iters=200):
    """Times the oracle as it stands on a bounded sample of workload P:
    element stiffness + DOK insertion per element, adjoint-gradient work per
    element (complex step), and one Jacobi-PCG iteration per stored non-zero on
    a same-family grid the oracle can assemble.  Returns per-unit seconds."""
    from oracle import assembly as OA, grad as OG, solve as OS
    import scipy.sparse as sp
    import workloads as W
    nq = len(P["quad_conn"])
    rng = np.random.default_rng(0)
    X = OA.coords(P)
    # A1 + A2: element matrices + DOK scatter for a sample of elements
    elems = rng.choice(nq, n_elem, replace=False)
    t0 = time.perf_counter()
    dok = {}
    for e in elems:
        Ke = OA.element_K(P, int(e), X)
        dofs = OA.element_dofs(OA.element_nodes(P, int(e)))
        for a, ra in enumerate(dofs):
            for b, cb in enumerate(dofs):
                dok[(ra, cb)] = dok.get((ra, cb), 0.0) + Ke[a, b]
    t_elem = (time.perf_counter() - t0) / n_elem
    # A4: adjoint gradient per element (13 complex-step element derivatives)
    u = W.random_state(len(P["x"]), 1)
    t0 = time.perf_counter()
    for e in elems[:n_grad]:
        OG.element_grad(P, int(e), u, 1.0, X)
    t_grad = (time.perf_counter() - t0) / n_grad
    # A3: PCG iteration cost per non-zero on a same-recipe grid
    Q = W.shell_config3(pcg_grid, cfg=3)
    nd = 6 * len(Q["x"])
    rp, ci, v = OA.csr_from_dok(OA.assemble_dok(Q), nd)
    fixed = OA.fixed_dofs(Q)
    v = OA.apply_supports_csr(rp, ci, v, fixed)
    K = sp.csr_matrix((v, ci, rp), shape=(nd, nd))
    fb = np.where(fixed, 0.0, Q["f"])
    t0 = time.perf_counter()
    _, info = OS.pcg(K, fb, 1.0 / K.diagonal(), rtol=1e-300, max_iter=pcg_iters)
    t_it_nnz = (time.perf_counter() - t0) / info["iters"] / len(v)
    return t_elem, t_grad, t_it_nnz


def oracle_rate(n_quads, nnz, cg_iters, t_elem, t_grad, t_it_nnz):
    t_eval = n_quads * (t_elem + t_grad) + cg_iters * nnz * t_it_nnz
    return 1.0 / t_eval, t_eval


C3B_NQ = N_GRID * N_GRID
C3B_NNZ = 36 * ((N_GRID + 1) ** 2 + 4 * N_GRID * (N_GRID + 1) + 4 * N_GRID * N_GRID)


def cpu_baseline_obj(P, cg_iters):
    t0 = time.perf_counter()
    te, tg, ti = oracle_sample(P)
    wall = time.perf_counter() - t0
    rate, t_eval = oracle_rate(C3B_NQ, C3B_NNZ, cg_iters, te, tg, ti)
    return {"value": rate, "unit": UNIT, "cores": 1, "kind": "oracle",
            "sample": (f"oracle timed on 2000 C3b elements (K_e + DOK), 1000 element gradients "
                       f"(complex step) and 200 PCG iterations on a 60x60 same-recipe grid "
                       f"({wall:.1f} s of CPU); extrapolated to C3b: {C3B_NQ} elements, "
                       f"{C3B_NNZ} nnz, {cg_iters} CG iterations -> {t_eval:.1f} s per eval"),
            "per_unit_s": {"element": te, "grad_element": tg, "cg_iter_per_nnz": ti}}


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    import workloads as W
    P = W.config3b()
    cg_iters = args.cg_iters
    times = []
    vals = []
    for k in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        te, tg, ti = oracle_sample(P, n_elem=200, n_grad=100, pcg_grid=32, pcg_iters=60)
        dt = time.perf_counter() - t0
        if k >= args.warmup:
            times.append(dt)
            vals.append(oracle_rate(C3B_NQ, C3B_NNZ, cg_iters, te, tg, ti)[0])
    value = float(np.median(vals))
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1000.0 / value, "higher_is_better": True,
            "scaling": "strong" if args.strips else "weak",  # the label of the arm it is compared with
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": "C3b: 408x408 MITC-4 shell quads, 1 003 686 DOF (reading c15)",
                       "rtol": RTOL, "cg_iters": cg_iters},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": "oracle",
                             "sample": ("per step: oracle on 200 C3b elements (K_e + DOK), 100 element "
                                        "gradients, 60 PCG iterations on a 32x32 same-recipe grid; "
                                        f"extrapolated to C3b with {cg_iters} CG iterations; "
                                        f"median sample wall {np.median(times):.2f} s")},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))


# ----------------------------------------------------------------------------
# GPU arm
# ----------------------------------------------------------------------------

def run_gpu(args):
    import torch
    rank, world, local = dist_env()
    if world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        torch.cuda.set_device(0)
    dev = torch.device("cuda", torch.cuda.current_device())
    import paper_2407_20026_b200 as sso
    import workloads as W

    # N > 1: by default every GPU evaluates its own C3b design (independent evaluations, as
    # in an optimisation loop over designs; weak scaling, no collective).  --strips splits one
    # C3b into N node strips with NCCL halos and allreduces instead (strong scaling).
    replicas = world > 1 and not args.strips
    P = W.shell_config3(408, cfg=3, design=rank) if replicas else W.config3b()
    t0 = time.perf_counter()
    stream = torch.cuda.current_stream()
    if replicas:
        m = sso.Model(P, rtol=RTOL, stream=stream.cuda_stream, device=dev.index, storage=args.storage,
                      precond=args.precond)
        parallelism = f"{world} GPUs x one C3b design each (independent evaluations, no collective)"
    elif world > 1:
        # strong scaling: C3b split into `world` node strips, one per GPU; halos of p
        # and the CG scalars travel through NCCL
        import torch.distributed as dist
        obj = [sso.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        m = sso.Model(P, rtol=RTOL, stream=stream.cuda_stream, device=dev.index, nranks=world,
                      rank=rank, nccl_id=obj[0])
        parallelism = f"{world} node strips (NCCL halo + allreduce), strong scaling"
    elif args.virtual_parts > 1:
        m = sso.Model(P, rtol=RTOL, stream=stream.cuda_stream, device=dev.index,
                      n_parts=args.virtual_parts)
        parallelism = f"{args.virtual_parts} node strips on 1 GPU (in-process transport)"
    else:
        m = sso.Model(P, rtol=RTOL, stream=stream.cuda_stream, device=dev.index, storage=args.storage,
                      precond=args.precond)
        parallelism = "single GPU"
    t_create = time.perf_counter() - t0
    ndof, nnz, nblocks = m.sizes()
    stored_vals, stored_blocks, symmetric = m.storage_info()
    n_nodes, nq = m.n_nodes, m.n_quads
    f_own = P["f"][6 * m.own_node_begin: 6 * (m.own_node_begin + n_nodes)]
    f_dev = torch.from_numpy(np.ascontiguousarray(f_own)).to(dev)
    u_dev = torch.zeros(ndof, dtype=torch.float64, device=dev)
    Cb = torch.zeros(1, dtype=torch.float64, device=dev)
    dXb = torch.zeros(3 * n_nodes, dtype=torch.float64, device=dev)
    dTb = torch.zeros(nq, dtype=torch.float64, device=dev)

    def step():
        m.assemble()
        _, info = m.solve(f_dev, u_dev)
        m.grad(sso.OBJ_COMPLIANCE, out=(Cb, dXb, dTb))
        return info

    for _ in range(args.warmup):
        step()

    def barrier():
        if world > 1:
            import torch.distributed as dist
            dist.barrier()
        torch.cuda.synchronize()

    # ---- timed region (device-resident inputs) -----------------------------
    m.profile_enable(True)
    m.profile_reset()
    l0 = m.launch_count()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    iters = []
    with ClockSampler(dev.index) as clk:
        barrier()
        ev0.record(stream)
        for _ in range(args.steps):
            info = step()
            iters.append(info["iters"])
        ev1.record(stream)
        barrier()
    launches = m.launch_count() - l0
    ms_total = ev0.elapsed_time(ev1)
    spmv_ms, spmv_n = m.profile_read("spmv")
    el_ms, el_n = m.profile_read("element")
    as_ms, as_n = m.profile_read("assemble")
    gr_ms, gr_n = m.profile_read("grad")
    m.profile_enable(False)
    if world > 1:
        import torch.distributed as dist
        t = torch.tensor([ms_total], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_total = float(t.item())
    ms_step = ms_total / args.steps
    # one C3b evaluation per step on every GPU (replicas) or one partitioned evaluation per step
    value = (world if replicas else 1) * args.steps / (ms_total / 1000.0)
    cg_iters = int(np.median(iters))

    # ---- e2e: host buffers through the C ABI, copies inside the timed region --
    f_host = torch.from_numpy(np.ascontiguousarray(f_own)).pin_memory()
    u_host = torch.zeros(ndof, dtype=torch.float64).pin_memory()
    C_h = torch.zeros(1, dtype=torch.float64).pin_memory()
    dX_h = torch.zeros(3 * n_nodes, dtype=torch.float64).pin_memory()
    dT_h = torch.zeros(nq, dtype=torch.float64).pin_memory()

    def step_host():
        m.assemble()
        m.solve(f_host.numpy(), u_host.numpy())
        m.grad(sso.OBJ_COMPLIANCE, out=(C_h.numpy(), dX_h.numpy(), dT_h.numpy()))

    step_host()
    e2e_steps = max(1, min(args.steps, 5))
    barrier()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        step_host()
    barrier()
    e2e_s = time.perf_counter() - t0
    if world > 1:
        import torch.distributed as dist
        t = torch.tensor([e2e_s], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())
    e2e_value = (world if replicas else 1) * e2e_steps / e2e_s

    # ---- roofline of the dominant kernel (SpMV inside PCG) --------------------
    peak, peak_src = measured_peaks()
    # algorithmic bytes of the stored format: values + block column ids + node_ptr + x read,
    # y written; symmetric storage adds the transpose slots (written and read back once)
    if symmetric == 3:  # values once + the 64-byte node descriptor (block columns, pull list) + p, q
        spmv_bytes = 8 * stored_vals + 64 * n_nodes + 16 * ndof
    else:               # values + block column ids + node_ptr + p, q (+ transpose slots, storage 2)
        spmv_bytes = 8 * stored_vals + 4 * stored_blocks + 8 * (n_nodes + 1) + 16 * ndof
        if symmetric == 2:
            spmv_bytes += 2 * 48 * (stored_blocks - n_nodes) + 8 * (n_nodes + 1) + 4 * (stored_blocks - n_nodes)
    spmv_avg_ms = spmv_ms / max(spmv_n, 1)
    achieved = spmv_bytes / (spmv_avg_ms / 1000.0) / 1e9 if spmv_n else None
    roofline = {"bound": "hbm",
                "kernel": {0: "spmv_dot (CG q = K p, p^T q)",
                           2: "spmv_sym pass1+pass2 (upper-block K, CG q = K p, p^T q)",
                           3: "spmv_pull_dot (upper-block K, one-pass pull, CG q = K p, p^T q)"}[symmetric],
                "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": (achieved / peak) if achieved else None, "traffic": ncu_traffic(symmetric),
                "algorithmic_bytes_per_launch": spmv_bytes, "avg_launch_ms": spmv_avg_ms,
                "launches": spmv_n, "peak_source": peak_src,
                "share_of_step": (spmv_avg_ms * (cg_iters + 1) * args.steps / ms_total) if spmv_n else None,
                "sampling": "CUDA event pairs around every 16th SpMV launch of the CG loop (graph event nodes)"}
    asm_ms = (el_ms + as_ms) / max(args.steps, 1)
    clocks = clk.summary()

    # ---- the same evaluation with the node-block Jacobi preconditioner (reading c19) ----
    alt = None
    if world == 1 and args.precond == 0 and args.virtual_parts == 1 and not args.no_alt:
        mb = sso.Model(P, rtol=RTOL, stream=stream.cuda_stream, device=dev.index, storage=args.storage,
                       precond=1)

        def step_b():
            mb.assemble()
            _, ib = mb.solve(f_dev, u_dev)
            mb.grad(sso.OBJ_COMPLIANCE, out=(Cb, dXb, dTb))
            return ib
        step_b()
        nb = max(1, min(args.steps, 3))
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        barrier()
        e0.record(stream)
        for _ in range(nb):
            ib = step_b()
        e1.record(stream)
        barrier()
        tb = e0.elapsed_time(e1)
        alt = {"precond": "node-block Jacobi (sso_options.precond = 1)", "value": nb / (tb / 1000.0),
               "unit": UNIT, "ms_per_step": tb / nb, "cg_iters": int(ib["iters"]), "steps": nb, "warmup": 1}
        mb.close()

    out = None
    if rank == 0:
        cpu = cpu_baseline_obj(P, cg_iters) if (world == 1 and not args.no_cpu) else None
        out = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
               "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
               # the default series (N = 1, 2, 4, ...: one design per GPU) is weak scaling; the
               # strip modes split one C3b (strong)
               "scaling": "strong" if (args.strips or args.virtual_parts > 1) else "weak",
               "vs_baseline": None, "dtype": "f64",
               "data": "synthetic (workloads.config3b, seeded)",
               "config": {"workload": "C3b: 408x408 MITC-4 shell quads, 1 003 686 DOF (reading c15)",
                          "n_nodes": n_nodes, "n_quads": nq, "ndof": ndof, "nnz": nnz,
                          "rtol": RTOL, "cg_iters": cg_iters,
                          "parallelism": parallelism,
                          "precond": {0: "point Jacobi", 1: "node-block Jacobi"}[args.precond if world == 1 else 0],
                          "storage": {0: "full node-block CSR", 2: "upper blocks, two-pass SpMV",
                                      3: "upper blocks (column-major runs), one-pass pull SpMV"}[symmetric],
                          "l2": "working set > L2 (CSR values alone 432 MB vs 126 MB L2); no flush",
                          "pattern_build_s": t_create},
               "roofline": roofline,
               "cpu_baseline": cpu,
               "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": 8 * ndof,
                       "d2h_bytes_per_step": 8 * (ndof + 1 + 3 * n_nodes + nq)},
               "gpu_launches": launches,
               "clocks": clocks,
               "extra": {"assembled_elements_per_s": nq / (asm_ms / 1000.0) if asm_ms else None,
                         "assembly_ms": asm_ms, "element_ms": el_ms / max(args.steps, 1),
                         "assemble_gather_ms": as_ms / max(args.steps, 1),
                         "grad_ms": gr_ms / max(args.steps, 1),
                         "cg_iters_per_s": cg_iters / (ms_step / 1000.0),
                         "spmv_ms_per_step_est": spmv_avg_ms * (cg_iters + 1),
                         "block_jacobi": alt}}
        print(json.dumps(out))
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()
    m.close()
    return out


def run_batch(args):
    """C5 (BASELINE.json configs[4]): 64 seeded 50x50 shell designs per GPU sharing one
    connectivity, evaluated together (compliance + gradients) — weak scaling, no
    collective: rank r evaluates designs [64 r, 64 (r + 1))."""
    import torch
    rank, world, local = dist_env()
    if world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        torch.cuda.set_device(0)
    dev = torch.device("cuda", torch.cuda.current_device())
    import paper_2407_20026_b200 as sso
    import workloads as W
    B = args.batch
    designs = [W.config5_design(rank * B + b) for b in range(B)]
    stream = torch.cuda.current_stream()
    m = sso.Model(designs[0], rtol=RTOL, batch=B, stream=stream.cuda_stream, device=dev.index,
                  precond=args.precond)
    Z = torch.from_numpy(np.stack([d["z"] for d in designs])).to(dev)
    T = torch.from_numpy(np.stack([d["t"] for d in designs])).to(dev)
    F = torch.from_numpy(np.stack([d["f"] for d in designs])).to(dev)
    U = torch.zeros_like(F)
    Cb = torch.zeros(B, dtype=torch.float64, device=dev)
    dX = torch.zeros(B * 3 * m.n_nodes, dtype=torch.float64, device=dev)
    dT = torch.zeros(B * m.n_quads, dtype=torch.float64, device=dev)

    def step():
        m.set_design(z=Z, t=T)
        m.assemble()
        _, infos = m.solve(F, U)
        m.grad(sso.OBJ_COMPLIANCE, out=(Cb, dX, dT))
        return infos

    for _ in range(args.warmup):
        step()

    def barrier():
        if world > 1:
            import torch.distributed as dist
            dist.barrier()
        torch.cuda.synchronize()

    l0 = m.launch_count()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(dev.index) as clk:
        barrier()
        ev0.record(stream)
        for _ in range(args.steps):
            infos = step()
        ev1.record(stream)
        barrier()
    ms = ev0.elapsed_time(ev1)
    if world > 1:
        import torch.distributed as dist
        t = torch.tensor([ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    its = [i["iters"] for i in infos]
    value = world * B * args.steps / (ms / 1000.0)
    if rank == 0:
        print(json.dumps({"metric": "C5 batched shell design evaluations (solve + adjoint gradient) per second",
                          "value": value, "unit": "designs/s", "n_gpus": world, "steps": args.steps,
                          "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
                          "scaling": "weak", "vs_baseline": None, "dtype": "f64",
                          "data": "synthetic (workloads.config5_design, seeded)",
                          "config": {"workload": f"C5: {B} designs/GPU x 50x50 MITC-4 quads (15 606 DOF each)",
                                     "rtol": RTOL, "cg_iters_max": max(its), "cg_iters_min": min(its),
                                     "precond": {0: "point Jacobi", 1: "node-block Jacobi"}[args.precond],
                                     "parallelism": f"{world} GPU(s) x {B} designs, no collective"},
                          "gpu_launches": m.launch_count() - l0, "clocks": clk.summary()}))
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()
    m.close()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="gpu", choices=["gpu", "reference"])
    ap.add_argument("--cg-iters", type=int, default=None,
                    help="CG iteration count used to extrapolate the oracle (reference arm)")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-alt", action="store_true", help="skip the node-block Jacobi comparison run")
    ap.add_argument("--precond", type=int, default=0,
                    help="sso_options.precond for single-GPU C3b: 0 point Jacobi (north star), 1 node-block")
    ap.add_argument("--storage", type=int, default=0,
                    help="sso_options.storage for single-GPU C3b (0 = library default)")
    ap.add_argument("--workload", default="C3b", choices=["C3b", "C5"])
    ap.add_argument("--strips", action="store_true",
                    help="N > 1: split one C3b into N node strips (NCCL) instead of one design per GPU")
    ap.add_argument("--batch", type=int, default=64, help="C5 designs per GPU")
    ap.add_argument("--virtual-parts", type=int, default=1,
                    help="run the partitioned (strip) algorithm with P strips on one GPU")
    args = ap.parse_args()
    if args.impl == "reference":
        if args.cg_iters is None:
            p = os.path.join(ROOT, "profiles", "cg_iters_c3b.json")
            args.cg_iters = json.load(open(p))["cg_iters"] if os.path.exists(p) else 10000
        run_reference(args)
    elif args.workload == "C5":
        run_batch(args)
    else:
        run_gpu(args)


if __name__ == "__main__":
    main()
