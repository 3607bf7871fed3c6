"""Benchmark: shell FEA solve + adjoint gradient evaluations per second at 1M DOF
(BASELINE.json metric; workload C3b = 408 x 408 MITC-4 quads, 1 003 686 DOF,
reading c15), one step = one full pass of the hot path: A1+A2 element
stiffness + assembly (sso_assemble), A3 Jacobi-PCG to rtol (sso_solve), A4
compliance + adjoint gradient (sso_grad).  A0 (pattern) runs once at create.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--workload C3b|C4|C5]
                  [--replicas] [--virtual-parts P] [--impl reference]

N > 1 runs under torchrun (one rank per GPU).  By default the workload is split
into N contiguous node strips, one per GPU: every CG iteration exchanges the halo
of u over NCCL (overlapped with the interior rows' SpMV) and performs ONE
allreduce of the CG scalars (single-reduction CG, csrc/cg_sr.cu) -- strong
scaling (north_star "rows and elements partitioned across
2/4/8 GPUs").  --replicas instead evaluates one seeded design per GPU
(independent evaluations, no collective; weak scaling).  --virtual-parts P runs
the partitioned algorithm with P strips on one GPU (in-process transport).
--workload C4 is the north star's 6 M DOF partitioned configuration; C5 the
batched design evaluation (64 designs per GPU).
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


FLOP_ASM = 12495.0   # fp64 flop per quad, fused assembly (ncu exact DFMA/DMUL/DADD counts, profiles/r01)
FLOP_GRAD = 37426.0  # fp64 flop per quad, forward-mode dual-number gradient (same source)


def fp64_peak_tflops():
    """DFMA peak measured on the box by tools/dfma_peak.cu (profiles/fp64_peak.json), else the
    value derived from the guide's unit counts (64 FMA/clk/SM x 148 SMs x 1.965 GHz x 2)."""
    p = os.path.join(ROOT, "profiles", "fp64_peak.json")
    if os.path.exists(p):
        with open(p) as fh:
            d = json.load(fh)
        return float(d["tflops"]), "measured (profiles/fp64_peak.json, tools/dfma_peak.cu)"
    return 37.2, "derived (64 DFMA/clk/SM x 148 SMs x 1.965 GHz)"


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

_WP = None


def _worker_init(workload):
    global _WP
    import workloads as W
    _WP = {"C3b": W.config3b, "C4": W.config4, "C5": lambda: W.config5_design(0)}[workload]()


def _worker_elems(elems):
    """A1 + A2 on a chunk of elements (K_e + dict-of-keys insertion) and nothing else."""
    from oracle import assembly as OA
    X = OA.coords(_WP)
    dok = {}
    for e in elems:
        Ke = OA.element_K(_WP, int(e), X)
        dofs = OA.element_dofs(OA.element_nodes(_WP, int(e)))
        for a, ra in enumerate(dofs):
            for b, cb in enumerate(dofs):
                dok[(ra, cb)] = dok.get((ra, cb), 0.0) + Ke[a, b]
    return len(elems)


def _worker_grads(elems):
    """A4 on a chunk of elements (13 complex-step element derivatives each)."""
    import workloads as W
    from oracle import assembly as OA, grad as OG
    X = OA.coords(_WP)
    u = W.random_state(len(_WP["x"]), 1)
    for e in elems:
        OG.element_grad(_WP, int(e), u, 1.0, X)
    return len(elems)


def host_cores():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def oracle_sample(workload, n_quads, cores, n_elem_per_core=250, n_grad_per_core=40, pcg_grid=60,
                  pcg_iters=200):
    """Times the oracle as it stands on a bounded sample of the workload, on `cores` host
    cores (SURVEY.md §8(d) "Oracle timing"): element stiffness + DOK insertion and the
    complex-step adjoint gradient over a multiprocessing.Pool of `cores` workers (chunks of
    seeded elements), and Jacobi-PCG iterations (scipy CSR SpMV, one thread) on a
    same-recipe grid the oracle can assemble.  Returns per-unit seconds (elements per
    second of the whole pool, PCG seconds per iteration per stored non-zero)."""
    import multiprocessing as mp
    from oracle import assembly as OA, solve as OS
    import scipy.sparse as sp
    import workloads as W
    rng = np.random.default_rng(0)
    n_elem, n_grad = n_elem_per_core * cores, n_grad_per_core * cores
    k = max(n_elem, n_grad)
    elems = rng.choice(n_quads, k, replace=k > n_quads)  # C5 has 2 500 quads: many host cores revisit some
    ctx = mp.get_context("fork")
    with ctx.Pool(cores, initializer=_worker_init, initargs=(workload,)) as pool:
        pool.map(_worker_elems, [elems[:1]] * cores)  # workers built their inputs
        t0 = time.perf_counter()
        pool.map(_worker_elems, np.array_split(elems[:n_elem], cores))
        t_elem = (time.perf_counter() - t0) / n_elem
        t0 = time.perf_counter()
        pool.map(_worker_grads, np.array_split(elems[:n_grad], cores))
        t_grad = (time.perf_counter() - t0) / n_grad
    Q = W.config5_design(0) if workload == "C5" else W.shell_config3(pcg_grid, cfg=3)
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


def grid_nnz(n):
    return 36 * ((n + 1) ** 2 + 4 * n * (n + 1) + 4 * n * n)


WORKLOADS = {"C3b": (408, "C3b: 408x408 MITC-4 shell quads, 1 003 686 DOF (reading c15)"),
             "C4": (1000, "C4: 1000x1000 MITC-4 shell quads, 6 012 006 DOF, edge y=0 clamped + 2 pinned corners")}


SMALL = {"C1": ("config1", "C1: grid-shell, 40 frame elements (25 nodes, 150 DOF), corners pinned"),
         "C2": ("config2", "C2: 20x20 MITC-4 shallow shell (441 nodes, 2 646 DOF), boundary pinned")}


def small_metric(workload):
    return f"{workload} solve+adjoint grad evals/sec (latency configuration)"


def oracle_full_eval(workload):
    """One complete evaluation by the oracle as it stands (not a sample): DOK assembly, supports,
    dense Cholesky solve, compliance and the complex-step adjoint gradient.  Returns seconds."""
    import workloads as W
    from oracle import grad as OG
    P = getattr(W, SMALL[workload][0])()
    t0 = time.perf_counter()
    u, _, _ = OG.evaluate(P, solver="cholesky")
    OG.compliance(P["f"], u)
    OG.adjoint_gradient(P, u)
    return time.perf_counter() - t0


def cpu_baseline_full(workload):
    dt = oracle_full_eval(workload)
    return {"value": 1.0 / dt, "unit": UNIT, "cores": 1, "kind": "oracle", "extrapolated": False,
            "sample": (f"one complete {workload} evaluation by the oracle as it stands (DOK assembly, dense "
                       f"Cholesky, complex-step adjoint gradient), single process: {dt:.2f} s")}


def cpu_baseline_obj(workload, cg_iters, cores=None):
    n = WORKLOADS[workload][0]
    cores = cores or host_cores()
    t0 = time.perf_counter()
    te, tg, ti = oracle_sample(workload, n * n, cores)
    wall = time.perf_counter() - t0
    rate, t_eval = oracle_rate(n * n, grid_nnz(n), cg_iters, te, tg, ti)
    return {"value": rate, "unit": UNIT, "cores": cores, "kind": "oracle",
            "sample": (f"oracle as it stands on {workload} (extrapolated, not a full run): {250 * cores} "
                       f"elements (K_e + DOK) and {40 * cores} element gradients (complex step) over a "
                       f"{cores}-process pool, 200 PCG iterations (scipy CSR, 1 thread) on a 60x60 "
                       f"same-recipe grid; {wall:.1f} s wall; scaled to {n * n} elements, "
                       f"{grid_nnz(n)} nnz, {cg_iters} CG iterations -> {t_eval:.1f} s per eval"),
            "extrapolated": True,
            "per_unit_s": {"element": te, "grad_element": tg, "cg_iter_per_nnz": ti}}


C5_N = 50


def cpu_baseline_c5(cg_iters, cores=None, n_elem_per_core=250, n_grad_per_core=40, pcg_iters=200):
    """Oracle baseline for C5 in designs/s: the C5 designs are independent, so each host core
    evaluates its own design — per-design time on one core (pool element rates x cores, the
    PCG sample is single-threaded already) and `cores` designs in flight."""
    cores = cores or host_cores()
    nq = C5_N * C5_N
    t0 = time.perf_counter()
    te, tg, ti = oracle_sample("C5", nq, cores, n_elem_per_core, n_grad_per_core, pcg_iters=pcg_iters)
    wall = time.perf_counter() - t0
    t_design = nq * (te + tg) * cores + cg_iters * grid_nnz(C5_N) * ti
    return {"value": cores / t_design, "unit": "designs/s", "cores": cores, "kind": "oracle",
            "sample": (f"oracle as it stands on C5 design 0 (extrapolated, not a full run): "
                       f"{n_elem_per_core * cores} elements (K_e + DOK) and {n_grad_per_core * cores} element "
                       f"gradients over a {cores}-process pool, {pcg_iters} PCG iterations (scipy CSR, 1 "
                       f"thread) on the design itself; {wall:.1f} s wall; scaled to {nq} elements, "
                       f"{grid_nnz(C5_N)} nnz, {cg_iters} CG iterations = {t_design:.1f} s per design on one "
                       f"core, {cores} designs in flight"),
            "extrapolated": True,
            "per_unit_s": {"element": te, "grad_element": tg, "cg_iter_per_nnz": ti}}


C5_METRIC = "C5 batched shell design evaluations (solve + adjoint gradient) per second"
C5_ITERS = 3400  # median CG iterations of the 64 seeded C5 designs at rtol 1e-10 (profiles/r02/bench_c5.json)


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    if args.workload in SMALL:
        times = []
        for k in range(args.warmup + args.steps):
            dt = oracle_full_eval(args.workload)
            if k >= args.warmup:
                times.append(dt)
        value = args.steps / sum(times)
        print(json.dumps({"impl": "reference", "metric": small_metric(args.workload), "value": value, "unit": UNIT,
                          "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000.0 / value,
                          "higher_is_better": True, "scaling": "weak" if world > 1 else "strong", "vs_baseline": None, "dtype": "f64",
                          "data": "synthetic", "config": {"workload": SMALL[args.workload][1]},
                          "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": "oracle",
                                           "extrapolated": False,
                                           "sample": f"{args.steps} complete {args.workload} evaluations by the oracle"},
                          "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}))
        return
    if args.workload == "C5":
        times, vals = [], []
        for k in range(args.warmup + args.steps):
            t0 = time.perf_counter()
            cb = cpu_baseline_c5(C5_ITERS, n_elem_per_core=40, n_grad_per_core=6, pcg_iters=60)
            if k >= args.warmup:
                times.append(time.perf_counter() - t0)
                vals.append(cb["value"])
        value = float(np.median(vals))
        cb["value"] = value
        print(json.dumps({"impl": "reference", "metric": C5_METRIC, "value": value, "unit": "designs/s",
                          "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
                          "ms_per_step": 1000.0 / value, "higher_is_better": True, "scaling": "weak",
                          "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                          "config": {"workload": f"C5: {args.batch} designs/GPU x 50x50 MITC-4 quads (15 606 DOF each)",
                                     "rtol": RTOL, "cg_iters": C5_ITERS},
                          "cpu_baseline": cb,
                          "e2e": {"value": value, "unit": "designs/s", "h2d_bytes_per_step": 0,
                                  "d2h_bytes_per_step": 0}}))
        return
    n, wname = WORKLOADS[args.workload if args.workload in WORKLOADS else "C3b"]
    cg_iters = args.cg_iters
    cores = host_cores()
    times = []
    vals = []
    for k in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        te, tg, ti = oracle_sample(args.workload if args.workload in WORKLOADS else "C3b", n * n, cores,
                                   n_elem_per_core=40, n_grad_per_core=6, pcg_grid=32, pcg_iters=60)
        dt = time.perf_counter() - t0
        if k >= args.warmup:
            times.append(dt)
            vals.append(oracle_rate(n * n, grid_nnz(n), cg_iters, te, tg, ti)[0])
    value = float(np.median(vals))
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1000.0 / value, "higher_is_better": True,
            # the label of the GPU arm it is compared with
            "scaling": "weak" if (world > 1 and args.replicas) else "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": wname, "rtol": RTOL, "cg_iters": cg_iters},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle",
                             "extrapolated": True,
                             "sample": (f"per step (extrapolated, not a full run): oracle on {40 * cores} "
                                        f"elements (K_e + DOK) and {6 * cores} element gradients over a "
                                        f"{cores}-process pool, 60 PCG iterations (scipy CSR, 1 thread) on "
                                        f"a 32x32 same-recipe grid; scaled to {args.workload} with "
                                        f"{cg_iters} CG iterations; median sample wall {np.median(times):.2f} s")},
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

    # N > 1: the workload split into N node strips over NCCL (strong scaling, the default);
    # --replicas: every GPU evaluates its own seeded design of the workload (weak scaling).
    replicas = world > 1 and (args.replicas or args.workload in SMALL)  # C1, C2: replicas only
    if args.workload in SMALL:  # latency configs (replicas only across GPUs)
        wname = SMALL[args.workload][1]
        P = getattr(W, SMALL[args.workload][0])()
    else:
        n_grid, wname = WORKLOADS[args.workload]
        cfg, sup = (4, "c4") if args.workload == "C4" else (3, "clamped_edges")
        P = W.shell_config3(n_grid, cfg=cfg, supports=sup, design=rank if replicas else 0)
    t0 = time.perf_counter()
    stream = torch.cuda.current_stream()
    if replicas:
        m = sso.Model(P, rtol=RTOL, stream=stream.cuda_stream, device=dev.index, storage=args.storage,
                      precond=args.precond)
        parallelism = f"{world} GPUs x one {args.workload} design each (independent evaluations, no collective)"
    elif world > 1:
        # strong scaling: the workload split into `world` node strips, one per GPU; halos of u
        # and one allreduce of the CG scalars per iteration through NCCL
        import torch.distributed as dist
        obj = [sso.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        m = sso.Model(P, rtol=RTOL, stream=stream.cuda_stream, device=dev.index, nranks=world,
                      rank=rank, nccl_id=obj[0], precond=args.precond)
        parallelism = (f"{world} node strips (NCCL halo overlapped with the interior SpMV, one allreduce "
                       f"per CG iteration), strong scaling")
    elif args.virtual_parts > 1:
        m = sso.Model(P, rtol=RTOL, stream=stream.cuda_stream, device=dev.index,
                      n_parts=args.virtual_parts, precond=args.precond)
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
    iters, solve_ms = [], []
    with ClockSampler(dev.index) as clk:
        barrier()
        ev0.record(stream)
        for _ in range(args.steps):
            info = step()
            iters.append(info["iters"])
            solve_ms.append(info["ms"])
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
    # algorithmic bytes of the stored format (per rank: its owned rows)
    if symmetric == 3:  # values once + the 64-byte node descriptor (block columns, pull list) + p, q
        spmv_bytes = 8 * stored_vals + 64 * n_nodes + 16 * ndof
    else:               # values + block column ids + node_ptr + p, q
        spmv_bytes = 8 * stored_vals + 4 * stored_blocks + 8 * (n_nodes + 1) + 16 * ndof
    spmv_avg_ms = spmv_ms / max(spmv_n, 1)
    achieved = spmv_bytes / (spmv_avg_ms / 1000.0) / 1e9 if spmv_n else None
    roofline = {"bound": "hbm",
                "kernel": {0: "spmv_dot (CG q = K p, p^T q)",
                           3: "spmv_pull_dot (upper-block K, one-pass pull, CG q = K p, p^T q)"}[symmetric],
                "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": (achieved / peak) if achieved else None, "traffic": ncu_traffic(symmetric),
                "algorithmic_bytes_per_launch": spmv_bytes, "avg_launch_ms": spmv_avg_ms,
                "launches": spmv_n, "peak_source": peak_src,
                "share_of_step": (spmv_avg_ms * (cg_iters + 1) * args.steps / ms_total) if spmv_n else None,
                "sampling": ("CUDA event pairs around every 16th SpMV launch of the CG loop (graph event nodes)"
                             + ("; one launch covers every strip" if args.virtual_parts > 1 else ""))}
    if args.workload in SMALL:
        # latency configuration: the CG loop runs in the persistent cluster kernel (cg_small.cu),
        # no per-iteration SpMV launch to sample; the figure that bounds it is the time per
        # iteration (3 cluster barriers + the row products), not bandwidth
        us_it = 1000.0 * float(np.median(solve_ms)) / max(cg_iters, 1)
        roofline = {"bound": "latency", "kernel": "cg_cluster_kernel (persistent cluster PCG, csrc/cg_small.cu)",
                    "achieved": us_it, "unit": "us/iteration", "peak": None, "frac": None, "traffic": None,
                    "note": "solve time (incl. init, true-residual check, Lanczos) / CG iterations, median of the "
                            "timed steps"}
    asm_ms = (el_ms + as_ms) / max(args.steps, 1)
    grad_ms = gr_ms / max(args.steps, 1)
    clocks = clk.summary()
    # assembly and gradient rooflines: HBM on the survey's algorithmic bytes
    # (CSR values written 8 nnz + dinv 8 DOF + coordinates 24 n + connectivity, t, rank map
    # 88 E) and on the bytes the stored format writes; fp64 on the exact instruction counts
    # (ncu, profiles/r01: 12 495 flop per quad assembled, 37 426 per quad gradient) against
    # the on-box DFMA microbenchmark (profiles/fp64_peak.json) when present
    fp64_peak, fp64_src = fp64_peak_tflops()
    asm_bytes_survey = 8 * nnz + 8 * ndof + 24 * n_nodes + 88 * nq
    asm_bytes_stored = (8 * 38 if symmetric == 3 else 8 * 36) * stored_blocks + 8 * ndof + 24 * n_nodes + 88 * nq
    grad_bytes = 8 * ndof + 48 * n_nodes + 32 * nq + 192 * nq
    rooflines = {
        "assembly": {"ms": asm_ms, "hbm_bytes_survey": asm_bytes_survey, "hbm_bytes_stored": asm_bytes_stored,
                     "hbm_frac_survey": asm_bytes_survey / (asm_ms / 1e3) / 1e9 / peak if asm_ms else None,
                     "hbm_frac_stored": asm_bytes_stored / (asm_ms / 1e3) / 1e9 / peak if asm_ms else None,
                     "flops": FLOP_ASM * nq, "fp64_frac": (FLOP_ASM * nq / (asm_ms / 1e3) / 1e12 / fp64_peak)
                     if asm_ms else None},
        "gradient": {"ms": grad_ms, "hbm_bytes": grad_bytes,
                     "hbm_frac": grad_bytes / (grad_ms / 1e3) / 1e9 / peak if grad_ms else None,
                     "flops": FLOP_GRAD * nq, "fp64_frac": (FLOP_GRAD * nq / (grad_ms / 1e3) / 1e12 / fp64_peak)
                     if grad_ms else None},
        "fp64_peak_tflops": fp64_peak, "fp64_peak_source": fp64_src, "hbm_peak_gbs": peak}

    # ---- the same evaluation with the node-block Jacobi preconditioner (reading c19) ----
    alt = None
    if world == 1 and args.precond == 0 and args.virtual_parts == 1 and not args.no_alt and args.workload == "C3b":
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
        cpu = None
        if world == 1 and not args.no_cpu:
            cpu = cpu_baseline_full(args.workload) if args.workload in SMALL else cpu_baseline_obj(args.workload, cg_iters)
        strong = (world > 1 and not replicas) or args.virtual_parts > 1 or (world == 1 and not args.replicas)
        out = {"metric": small_metric(args.workload) if args.workload in SMALL else METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
               "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
               # the default series (N = 1, 2, 4, 8) splits one workload into N strips: strong
               "scaling": "strong" if strong else "weak",
               "vs_baseline": None, "dtype": "f64",
               "data": f"synthetic (workloads.shell_config3 {args.workload} recipe, seeded)",
               "config": {"workload": wname,
                          "n_nodes_per_rank": n_nodes, "n_quads_per_rank": nq, "ndof_per_rank": ndof, "nnz": nnz,
                          "rtol": RTOL, "cg_iters": cg_iters,
                          "parallelism": parallelism,
                          "precond": {0: "point Jacobi", 1: "node-block Jacobi"}[args.precond],
                          "storage": {0: "full node-block CSR",
                                      3: "upper blocks (38-double 2x2 sub-block records), one-pass pull SpMV"}[symmetric],
                          "l2": ("working set > L2 (CSR values >= 254 MB vs 126 MB L2); no flush"
                                 if args.workload not in SMALL else
                                 "working set < L2 (a latency configuration; no flush)"),
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
                         "grad_ms": grad_ms,
                         "cg_iters_per_s": cg_iters / (ms_step / 1000.0),
                         "spmv_ms_per_step_est": spmv_avg_ms * (cg_iters + 1),
                         "rooflines": rooflines,
                         "certification": {k: info.get(k) for k in ("true_rel_res", "lanczos_iters", "lanczos_lmin",
                                                                      "lanczos_lmax", "err_energy_est", "err2_est")},
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

    m.profile_enable(True)
    m.profile_reset()
    l0 = m.launch_count()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(dev.index) as clk:
        barrier()
        ev0.record(stream)
        for _ in range(args.steps):
            infos = step()
        ev1.record(stream)
        barrier()
    launches = m.launch_count() - l0
    ms = ev0.elapsed_time(ev1)
    spmv_ms, spmv_n = m.profile_read("spmv")
    m.profile_enable(False)
    if world > 1:
        import torch.distributed as dist
        t = torch.tensor([ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    its = [i["iters"] for i in infos]
    value = world * B * args.steps / (ms / 1000.0)

    # e2e: host (pinned) design arrays and loads in, u / C / gradients out, every step
    Zh, Th, Fh = Z.cpu().pin_memory(), T.cpu().pin_memory(), F.cpu().pin_memory()
    Uh = torch.zeros_like(Fh).pin_memory()
    Ch = torch.zeros(B, dtype=torch.float64).pin_memory()
    dXh = torch.zeros(B * 3 * m.n_nodes, dtype=torch.float64).pin_memory()
    dTh = torch.zeros(B * m.n_quads, dtype=torch.float64).pin_memory()

    def step_host():
        m.set_design(z=Zh.numpy(), t=Th.numpy())
        m.assemble()
        m.solve(Fh.numpy(), Uh.numpy())
        m.grad(sso.OBJ_COMPLIANCE, out=(Ch.numpy(), dXh.numpy(), dTh.numpy()))

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

    # roofline of the batched SpMV (one launch covers all B designs)
    peak, peak_src = measured_peaks()
    ndof = m.ndof
    stored_vals, stored_blocks, symmetric = m.storage_info()
    # values and p, q per design; the shared pattern (node descriptors / block columns) once
    per_design = 8 * stored_vals + 16 * ndof
    shared = 64 * m.n_nodes if symmetric == 3 else 4 * stored_blocks + 8 * (m.n_nodes + 1)
    spmv_bytes = B * per_design + shared
    spmv_avg_ms = spmv_ms / max(spmv_n, 1)
    achieved = spmv_bytes / (spmv_avg_ms / 1000.0) / 1e9 if spmv_n else None
    roofline = {"bound": "hbm", "kernel": "batched SpMV of the CG loop (all designs in one launch)",
                "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak if achieved else None, "traffic": None,
                "algorithmic_bytes_per_launch": spmv_bytes, "avg_launch_ms": spmv_avg_ms,
                "launches": spmv_n, "peak_source": peak_src,
                "share_of_step": (spmv_avg_ms * (max(its) + 1) * args.steps / ms) if spmv_n else None,
                "sampling": "CUDA event pairs around every 16th SpMV launch of the CG loop (graph event nodes)"}
    if rank == 0:
        cpu = cpu_baseline_c5(int(np.median(its))) if (world == 1 and not args.no_cpu) else None
        print(json.dumps({"metric": C5_METRIC,
                          "value": value, "unit": "designs/s", "n_gpus": world, "steps": args.steps,
                          "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
                          "scaling": "weak", "vs_baseline": None, "dtype": "f64",
                          "data": "synthetic (workloads.config5_design, seeded)",
                          "config": {"workload": f"C5: {B} designs/GPU x 50x50 MITC-4 quads (15 606 DOF each)",
                                     "rtol": RTOL, "cg_iters_max": max(its), "cg_iters_min": min(its),
                                     "precond": {0: "point Jacobi", 1: "node-block Jacobi"}[args.precond],
                                     "parallelism": f"{world} GPU(s) x {B} designs, no collective",
                                     "storage": {0: "full node-block CSR", 3: "upper blocks (38-double records), "
                                                 "one-pass pull SpMV"}[symmetric],
                                     "l2": f"working set {spmv_bytes / 1e6:.0f} MB per SpMV vs 126 MB L2; no flush"},
                          "roofline": roofline, "cpu_baseline": cpu,
                          "e2e": {"value": world * B * e2e_steps / e2e_s, "unit": "designs/s",
                                  "h2d_bytes_per_step": 8 * (Z.numel() + T.numel() + F.numel()),
                                  "d2h_bytes_per_step": 8 * (U.numel() + B + dX.numel() + dT.numel())},
                          "gpu_launches": launches, "clocks": clk.summary()}))
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
    ap.add_argument("--workload", default="C3b", choices=["C1", "C2", "C3b", "C4", "C5"])
    ap.add_argument("--replicas", action="store_true",
                    help="N > 1: one seeded design per GPU (independent, no collective) instead of N strips")
    ap.add_argument("--batch", type=int, default=64, help="C5 designs per GPU")
    ap.add_argument("--virtual-parts", type=int, default=1,
                    help="run the partitioned (strip) algorithm with P strips on one GPU")
    args = ap.parse_args()
    if args.impl == "reference":
        if args.cg_iters is None:
            p = os.path.join(ROOT, "profiles", "cg_iters_c3b.json")
            d = json.load(open(p)) if os.path.exists(p) else {}
            args.cg_iters = (d.get("cg_iters_" + args.workload, d.get("cg_iters", 10000))
                             if args.workload in WORKLOADS else 0)
        run_reference(args)
    elif args.workload == "C5":
        run_batch(args)
    else:
        run_gpu(args)


if __name__ == "__main__":
    main()
