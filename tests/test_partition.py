"""Host-side partition logic — CPU only, no GPU.

* Strip-local CSR patterns (sso_local_pattern) concatenate to the oracle's
  global DOK pattern bit-exactly, for even and uneven strips, beams and shells.
* Halo plans (sso_halo_plan) are consistent: the halo of a strip is exactly the
  set of non-owned nodes of elements touching it, and what strip q sends to p is
  exactly p's halo nodes owned by q, in p's halo order.
* world_size-2 gloo run: each rank builds its plan through the C ABI, exchanges
  the owned values of a seeded global vector with torch.distributed send/recv
  following the plan, and checks its received halo against the global vector;
  rank 0 checks the gathered local patterns against the oracle pattern.
"""
import os
import socket

import numpy as np
import pytest

import workloads as W
from oracle import assembly as OA


def mixed():
    P = W.tiny_shell(4, seed=3)
    P["beam_conn"] = np.array([[0, 6], [6, 12], [3, 9], [20, 24]], np.int32)
    nb = len(P["beam_conn"])
    P["A"], P["Iy"], P["Iz"], P["J"] = (np.full(nb, 1e-3), np.full(nb, 2e-6), np.full(nb, 1e-6),
                                        np.full(nb, 2e-6))
    P["E"] = np.concatenate([np.full(nb, 210e9), P["E"]])
    P["nu"] = np.concatenate([np.full(nb, 0.3), P["nu"]])
    return P


CASES = {
    "C2-2": (W.config2, [0, 220, 441]),
    "C2-3uneven": (W.config2, [0, 50, 300, 441]),
    "mixed-4": (mixed, [0, 5, 11, 19, 25]),
    "beams-2": (W.config1, [0, 12, 25]),
}


def oracle_pattern(P):
    nd = 6 * len(P["x"])
    rp, ci, _ = OA.csr_from_dok(OA.assemble_dok(P), nd)
    return rp, ci


@pytest.mark.parametrize("name", list(CASES))
def test_local_patterns_concatenate(name):
    import paper_2407_20026_b200 as sso
    make, ranges = CASES[name]
    P = make()
    rp, ci = oracle_pattern(P)
    rows, cols = [np.zeros(1, np.int64)], []
    base = 0
    for p in range(len(ranges) - 1):
        lrp, lci = sso.local_pattern(P, ranges, p)
        rows.append(lrp[1:] + base)
        cols.append(lci)
        base += lrp[-1]
    assert np.array_equal(np.concatenate(rows), rp)
    assert np.array_equal(np.concatenate(cols), ci)


def brute_halo(P, ranges, p):
    b, e = ranges[p], ranges[p + 1]
    halo = set()
    conns = [P["beam_conn"], P["quad_conn"]]
    for conn in conns:
        for el in conn:
            if any(b <= n < e for n in el):
                halo |= {int(n) for n in el if not (b <= n < e)}
    return sorted(halo)


@pytest.mark.parametrize("name", list(CASES))
def test_halo_plans_consistent(name):
    import paper_2407_20026_b200 as sso
    make, ranges = CASES[name]
    P = make()
    nparts = len(ranges) - 1
    plans = [sso.halo_plan(P, ranges, p) for p in range(nparts)]
    for p, (halo, sends) in enumerate(plans):
        assert halo.tolist() == brute_halo(P, ranges, p)
        for q, sent in sends.items():
            hq = plans[q][0]
            want = [g for g in hq if ranges[p] <= g < ranges[p + 1]]
            assert sent.tolist() == want


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    try:
        import torch
        import torch.distributed as dist
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        import paper_2407_20026_b200 as sso
        P = W.config2()
        n = len(P["x"])
        ranges = [0, 230, n]
        halo, sends = sso.halo_plan(P, ranges, rank)
        g = np.random.default_rng(11).standard_normal(6 * n)
        # send owned values to each neighbour, receive my halo from each owner
        reqs = []
        for nb, ids in sends.items():
            buf = torch.from_numpy(np.concatenate([g[6 * i:6 * i + 6] for i in ids]))
            reqs.append(dist.isend(buf, dst=nb))
        got = np.zeros(6 * len(halo))
        owners = np.searchsorted(np.asarray(ranges), halo, side="right") - 1
        for nb in sorted(set(owners.tolist())):
            sel = np.nonzero(owners == nb)[0]
            buf = torch.zeros(6 * len(sel), dtype=torch.float64)
            dist.recv(buf, src=nb)
            for k, i in enumerate(sel):
                got[6 * i:6 * i + 6] = buf[6 * k:6 * k + 6].numpy()
        for r in reqs:
            r.wait()
        want = np.concatenate([g[6 * h:6 * h + 6] for h in halo])
        ok_halo = bool(np.array_equal(got, want))
        rp, ci = sso.local_pattern(P, ranges, rank)
        gathered = [None] * world
        dist.all_gather_object(gathered, (rp, ci))
        ok_pat = True
        if rank == 0:
            orp, oci = oracle_pattern(P)
            rows, cols, base = [np.zeros(1, np.int64)], [], 0
            for lrp, lci in gathered:
                rows.append(lrp[1:] + base)
                cols.append(lci)
                base += lrp[-1]
            ok_pat = np.array_equal(np.concatenate(rows), orp) and np.array_equal(np.concatenate(cols), oci)
        dist.destroy_process_group()
        q.put((rank, ok_halo, ok_pat, ""))
    except Exception as e:  # pragma: no cover - reported to the parent
        q.put((rank, False, False, repr(e)))


def test_gloo_two_rank_halo_exchange():
    import multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    for rank, ok_halo, ok_pat, err in res:
        assert not err, err
        assert ok_halo, f"rank {rank}: halo values differ"
        assert ok_pat, f"rank {rank}: concatenated local patterns differ from the oracle"
