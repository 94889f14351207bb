"""torchrun: per-op graph timings of the distributed MLMG (C4 layout)."""
import os, sys, numpy as np, torch, torch.distributed as dist
sys.path.insert(0, '/root/repo')
world = int(os.environ.get("WORLD_SIZE", "1")); rank = int(os.environ.get("RANK", "0")); local = int(os.environ.get("LOCAL_RANK", "0"))
torch.cuda.set_device(local)
dist.init_process_group("nccl", device_id=torch.device("cuda", local))
import paper_2009_12009_b200 as A
from paper_2009_12009_b200 import stencil as S
f = {1: (1, 1, 1), 2: (2, 1, 1), 4: (2, 2, 1), 8: (2, 2, 2)}[world]
ext = tuple(256 * x for x in f)
dom = A.Box((0, 0, 0), tuple(e - 1 for e in ext))
ba = A.BoxArray([dom]).max_size(64)
dm = A.sfc_distribute(ba, A.default_costs(ba), world)
tr = A.Transport.distributed()
geom = A.Geometry(dom, (0.0,) * 3, tuple(e / 256.0 for e in ext), True)
mg = A.MLMG(geom, ba, dm, transport=tr, cluster_tail=int(os.environ.get('MB_CLUSTER', '2')),
           grid_level_cells=int(os.environ['MB_GRID']) if 'MB_GRID' in os.environ else None)
for lv in mg.levels:
    for fa in lv.phi: fa.storage.normal_()
    lv.rhs.storage.normal_()
top = mg.levels[0]
def graph_time(fn, reps=20):
    fn(); torch.cuda.synchronize(); dist.barrier(device_ids=[local])
    g = torch.cuda.CUDAGraph(); s = torch.cuda.Stream(); s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s, capture_error_mode="relaxed"):
            for _ in range(reps): fn()
    torch.cuda.current_stream().wait_stream(s); torch.cuda.synchronize(); dist.barrier(device_ids=[local])
    ts = []
    for _ in range(5):
        dist.barrier(device_ids=[local]); torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); g.replay(); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1) * 1e3 / reps)
    t = torch.tensor([np.median(ts)], device="cuda"); dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return t.item()
res = {}
res["peer_barrier"] = graph_time(lambda: tr.peer_barrier())
res["fill L0 w2"] = graph_time(lambda: mg._fill(top, top.phi[top.cur], 2))
res["fill L0 w1"] = graph_time(lambda: mg._fill(top, top.phi[top.cur], 1))
def sw():
    mg._sweep(top)
res["sweep L0 (+fill w2)"] = graph_time(sw)
res["resid_restrict L0"] = graph_time(lambda: mg._resid_restrict(0))
res["residual_norm"] = graph_time(lambda: mg._residual_norm())
nrm = torch.zeros(1, dtype=torch.float64, device="cuda")
res["sweep+norm L0 (+fill w2)"] = graph_time(lambda: mg._sweep(top, norm=nrm))
for l in range(1, len(mg.levels)):
    lv = mg.levels[l]
    if lv.replicated: break
    res[f"fill L{l} w2"] = graph_time(lambda: mg._fill(lv, lv.phi[lv.cur], 2))
L1 = mg.levels[1]
res["sweep L1 (+fill w2)"] = graph_time(lambda: mg._sweep(L1))
res["resid_restrict L1 (+gather)"] = graph_time(lambda: mg._resid_restrict(1))
res["prolong_sweep L0"] = graph_time(lambda: mg._prolong_sweep(0) if mg.levels[0].fuse else mg._prolong(0))
res["prolong_sweep L1"] = graph_time(lambda: mg._prolong_sweep(1) if L1.fuse else mg._prolong(1))
for l in range(mg.grid_from, mg.tail):
    res[f"level_grid L{l} down"] = graph_time(lambda: mg._level_grid(l, False))
    res[f"level_grid L{l} up"] = graph_time(lambda: mg._level_grid(l, True))
for l in range(2, mg.grid_from):
    lv = mg.levels[l]
    res[f"sweep L{l} (+fill w2)"] = graph_time(lambda: mg._sweep(lv))
res["coarse tail"] = graph_time(lambda: mg._coarse_tail())
mg._prime()
res["iteration (cycle + fused norm)"] = graph_time(lambda: mg._body(), 5)
if rank == 0:
    print("levels:", [(tuple(l.domain.extents()), l.replicated) for l in mg.levels], "grid_from", mg.grid_from,
          "tail", mg.tail, "cluster", mg.cluster_tail)
    for k, v in res.items(): print(f"world={world} {k:24s} {v:9.1f} us")
dist.barrier(device_ids=[local])
