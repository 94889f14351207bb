"""Host-side logic of the one-process-per-GPU path, exercised with 2, 4 and 8
gloo ranks on CPU: every rank derives the same plans and the same per-rank layouts, the
per-pair message sizes a sender computes equal what the receiver expects,
re-boxing per rank is consistent, and each rank's resident set is its owned
boxes.  (Device work is covered by tests/dist_check.py on GPUs.)"""

import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    if root not in sys.path:
        sys.path.insert(0, root)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2009_12009_b200 as A
    from paper_2009_12009_b200.mlmg import mg_hierarchy, rebox_per_rank

    # the weak-scaling shapes of C4 (bench.py _domain_for), scaled down
    ext = {2: (64, 32, 32), 4: (64, 64, 32), 8: (64, 64, 64)}[world]
    dom = A.Box((0, 0, 0), tuple(e - 1 for e in ext))
    ba = A.BoxArray([dom]).max_size(16)
    dm = A.sfc_distribute(ba, A.default_costs(ba), world)
    plan = A.build_plan_fill_boundary(ba, 2, dom, True)
    t = plan.table()
    # per ordered pair: cells sent by src rank, as the sender computes them
    sends = {}
    recvs = {}
    for row in t:
        s, d = dm[int(row[0])], dm[int(row[1])]
        if s == d:
            continue
        cells = int(np.prod(row[5:8] - row[2:5] + 1))
        if s == rank:
            sends[d] = sends.get(d, 0) + cells
        if d == rank:
            recvs[s] = recvs.get(s, 0) + cells
    allsends = [None] * world
    dist.all_gather_object(allsends, sends)
    ok = all(allsends[s].get(rank, 0) == recvs.get(s, 0) for s in range(world))
    # identical plans everywhere
    tabs = [None] * world
    dist.all_gather_object(tabs, t.tolist())
    ok &= all(x == tabs[0] for x in tabs)
    # re-boxing: one rectangular box per rank, owners preserved
    rba, rdm = rebox_per_rank(ba, dm)
    ok &= len(rba) == world and sorted(rdm.owner) == list(range(world))
    ok &= sum(b.num_cells() for b in rba) == dom.num_cells()
    # every rank box is one SFC octant / slab of the domain
    split = {2: (2, 1, 1), 4: (2, 2, 1), 8: (2, 2, 2)}[world]
    ok &= all(tuple(b.extents()) == tuple(e // f for e, f in zip(ext, split)) for b in rba)
    levels = [(tuple(d.lo), tuple(d.hi), k) for d, _, k in mg_hierarchy(dom, rba, nranks=world)]
    alllv = [None] * world
    dist.all_gather_object(alllv, levels)
    ok &= all(x == alllv[0] for x in alllv)
    # the same resolutions as the oracle's hierarchy on the user's layout
    from oracle import mlmg_ref as R

    want = [d for d, _, _ in R.mg_levels(((0, 0, 0), tuple(e - 1 for e in ext)),
                                          [(tuple(b.lo), tuple(b.hi)) for b in ba])]
    ok &= [(lo, hi) for lo, hi, _ in levels] == want
    # the rebox fill plan's remote pairs are the SFC neighbours: a message per ordered pair
    rplan = A.build_plan_fill_boundary(rba, 2, dom, True).table()
    pairs = {(rdm[int(r[0])], rdm[int(r[1])]) for r in rplan if rdm[int(r[0])] != rdm[int(r[1])]}
    expect = {2: 2, 4: 12, 8: 56}[world]
    ok &= len(pairs) == expect
    # distributed FabArray on CPU storage: resident set = owned boxes (layout only)
    fa = A.FabArray(ba, dm, 1, 1, device="cpu")
    ok &= fa.distributed and set(fa.fabs) == set(dm.owned_indices(rank))
    gt = fa.global_fabtab()
    mine = dm.owned_indices(rank)
    ok &= bool(np.array_equal(gt[mine], fa.fabtab[mine]))
    out[rank] = bool(ok)
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4, 8])
def test_multi_rank_host_logic(world):
    port = _free_port()
    ctx = mp.get_context("spawn")
    mgr = ctx.Manager()
    out = mgr.dict()
    procs = [ctx.Process(target=_worker, args=(r, world, port, out)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
    assert all(p.exitcode == 0 for p in procs)
    assert dict(out) == {r: True for r in range(world)}
