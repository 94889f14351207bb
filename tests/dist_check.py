"""Multi-GPU check (run with torchrun, one process per GPU).

Solves the same periodic Poisson problem (a) distributed over all ranks with
NCCL ghost exchange and (b) on rank 0 alone, and checks that both give the
same iteration count, residual history and bit-identical solution.  Also
checks fill_boundary / parallel_copy / reduce over NCCL against a single-rank
run on rank 0.
"""

import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2009_12009_b200 as A  # noqa: E402


def main():
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    rank, world = dist.get_rank(), dist.get_world_size()
    def say(*m):
        if os.environ.get("DIST_VERBOSE"):
            print(f"[rank {rank}]", *m, flush=True)

    say("init")
    tr = A.Transport.distributed()
    say("nccl comm up")
    n = int(os.environ.get("DIST_N", "64"))
    ext = {1: (1, 1, 1), 2: (2, 1, 1), 4: (2, 2, 1), 8: (2, 2, 2)}[world]
    shape = tuple(n * e for e in ext)
    dom = A.Box((0, 0, 0), tuple(s - 1 for s in shape))
    ba = A.BoxArray([dom]).max_size(n // 2)
    dmw = A.sfc_distribute(ba, A.default_costs(ba), world)
    # weak scaling: the physical domain grows with the grid, cells stay cubic
    geom = A.Geometry(dom, (0.0,) * 3, tuple(float(e) for e in ext), True)
    rng = np.random.default_rng(7)
    g = rng.standard_normal(shape)
    g -= g.mean()
    ok = True

    # -- fill_boundary over NCCL vs single rank (rank 0) -------------------------
    fa = A.MultiFab(ba, dmw, 2, 2)
    gg = rng.standard_normal((2,) + shape)
    fa.setval(-7777.0)
    fa.load_valid_from(dom, gg)
    A.fill_boundary(fa, tr, dom, True)
    torch.cuda.synchronize()
    say("fill done")
    mine = {i: f.data.cpu().numpy() for i, f in fa.fabs.items()}
    allv = [None] * world
    dist.all_gather_object(allv, mine)
    red = [A.reduce(fa, k, 1, tr) for k in ("sum", "min", "max")]
    say("reduce done", red)
    if rank == 0:
        d1 = A.DistributionMapping.single_rank(len(ba))
        fb = A.MultiFab(ba, d1, 2, 2)
        fb.setval(-7777.0)
        fb.load_valid_from(dom, gg)
        A.fill_boundary(fb, A.Transport(1), dom, True)
        merged = {}
        for part in allv:
            merged.update(part)
        for i, f in fb.fabs.items():
            if not np.array_equal(merged[i], f.data.cpu().numpy()):
                print(f"FILL MISMATCH box {i}", flush=True)
                ok = False
        r1 = [A.reduce(fb, k, 1, A.Transport(1)) for k in ("sum", "min", "max")]
        if not (np.isclose(red[0], r1[0], rtol=1e-12) and red[1:] == r1[1:]):
            print("REDUCE MISMATCH", red, r1, flush=True)
            ok = False

    # -- MLMG distributed vs single rank ----------------------------------------------
    rhs = A.MultiFab(ba, dmw, 1, 0)
    rhs.load_valid_from(dom, g)
    phi = A.MultiFab(ba, dmw, 1, 1)
    mg = A.MLMG(geom, ba, dmw, transport=tr, use_graph=os.environ.get("DIST_GRAPH", "1") == "1")
    say("mlmg built", [(lv.kind, len(lv.ba)) for lv in mg.levels], "tail", mg.tail)
    rn = mg.solve(phi, rhs, rtol=1e-10, max_iter=60)
    say("solve done", mg.iterations)
    # a second solve on the same solver (graph replay) reproduces the first
    hist1 = list(mg.history)
    phi_again = A.MultiFab(ba, dmw, 1, 1)
    mg.solve(phi_again, rhs, rtol=1e-10, max_iter=60)
    same_again = mg.history == hist1 and all(torch.equal(phi.fab(i).valid(), phi_again.fab(i).valid())
                                             for i in phi.fabs)
    flag = torch.tensor([1 if same_again else 0], device="cuda")
    dist.all_reduce(flag, op=dist.ReduceOp.MIN)
    if rank == 0:
        print(f"repeated solve identical={bool(flag.item())}", flush=True)
    ok = ok and bool(flag.item())
    mine = {i: f.valid().cpu().numpy() for i, f in phi.fabs.items()}
    allv = [None] * world
    dist.all_gather_object(allv, mine)
    if rank == 0:
        d1 = A.DistributionMapping.single_rank(len(ba))
        r1 = A.MultiFab(ba, d1, 1, 0)
        r1.load_valid_from(dom, g)
        p1 = A.MultiFab(ba, d1, 1, 1)
        m1 = A.MLMG(geom, ba, d1, transport=A.Transport(1))
        rn1 = m1.solve(p1, r1, rtol=1e-10, max_iter=60)
        merged = {}
        for part in allv:
            merged.update(part)
        same = all(np.array_equal(merged[i], f.valid().cpu().numpy()) for i, f in p1.fabs.items())
        print(f"world={world} dist iters={mg.iterations} single iters={m1.iterations} "
              f"hist_equal={mg.history == m1.history} phi_bit_identical={same} rn={rn:.3e} rn1={rn1:.3e}",
              flush=True)
        ok = ok and same and mg.history == m1.history

    # -- the same solve with the other ghost exchanges ----------------------------------
    # (default: p2p fills; True: every ghost pushed by the sweeps; "remote":
    # cross-GPU faces pushed, same-GPU records copied by the barrier fill)
    if tr.p2p:
        for variant in (True, "remote", "pull", "nogrid"):
            phi2 = A.MultiFab(ba, dmw, 1, 1)
            if variant == "pull":  # sweeps copy their input's ghosts themselves
                mg2 = A.MLMG(geom, ba, dmw, transport=tr, ghost_pull=True)
            elif variant == "nogrid":  # replicated levels as streaming sweeps + wrap fills (the 8-GPU 128^3 level)
                mg2 = A.MLMG(geom, ba, dmw, transport=tr, grid_level_cells=0)
            else:
                mg2 = A.MLMG(geom, ba, dmw, transport=tr, ghost_push=variant)
            pushing = any((lv.push is not None and lv.push[0].remote) or (lv.pull is not None and lv.pull[0].remote)
                          for lv in mg2.levels)
            mg2.solve(phi2, rhs, rtol=1e-10, max_iter=60)
            same2 = all(torch.equal(phi.fab(i).valid(), phi2.fab(i).valid()) for i in phi.fabs)
            flag = torch.tensor([1 if (same2 and mg2.history == mg.history) else 0], device="cuda")
            dist.all_reduce(flag, op=dist.ReduceOp.MIN)
            if rank == 0:
                print(f"ghost exchange {variant}: remote={pushing} identical={bool(flag.item())}", flush=True)
                ok = ok and bool(flag.item())

    # -- max-all-reduce over NVLink: values and NaN propagation -----------------------
    if tr.p2p:
        t = torch.tensor([float(rank + 1)], dtype=torch.float64, device="cuda")
        tr.peer_allmax(t)
        nan = torch.tensor([float("nan") if rank == world - 1 else 1.0], dtype=torch.float64, device="cuda")
        tr.peer_allmax(nan)
        torch.cuda.synchronize()
        good = t.item() == float(world) and bool(torch.isnan(nan).item())
        flag = torch.tensor([1 if good else 0], device="cuda")
        dist.all_reduce(flag, op=dist.ReduceOp.MIN)
        if rank == 0:
            print(f"peer_allmax: max={t.item()} nan_propagates={bool(torch.isnan(nan).item())} ok={bool(flag.item())}",
                  flush=True)
            ok = ok and bool(flag.item())

    # -- failure detection: a peer that never arrives ---------------------------------
    if tr.p2p:
        from paper_2009_12009_b200._native import set_option

        set_option("peer_timeout_ms", 300)
        dist.barrier()
        if rank == 0:
            import time

            t0 = time.time()
            tr.peer_barrier()  # rank 1 never joins this one
            torch.cuda.synchronize()
            try:
                tr.check_faults()
                print("STALL NOT DETECTED", flush=True)
                ok = False
            except A.TransportError as e:
                print(f"stalled peer detected after {time.time() - t0:.2f} s: {e}", flush=True)
        dist.barrier()
    if rank == 0:
        print("DIST_CHECK", "PASS" if ok else "FAIL", flush=True)
    dist.barrier()
    if rank == 0 and not ok:
        sys.exit(1)


if __name__ == "__main__":
    main()
