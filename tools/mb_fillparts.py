"""torchrun: the p2p fill of the C4 fine level split into its parts."""
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
mg = A.MLMG(geom, ba, dm, transport=tr)
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
f = top.phi[0]
res["peer_barrier"] = graph_time(lambda: tr.peer_barrier())
res["p2p fill w2"] = graph_time(lambda: A.fill_boundary(f, tr, top.domain, True, ngrow=2, _post_barrier=False))
res["local-sources fill w2 + barrier"] = graph_time(lambda: A.fill_boundary(f, tr, top.domain, True, ngrow=2, _post_barrier=False, _local_sources=True))
res["p2p fill w1"] = graph_time(lambda: A.fill_boundary(f, tr, top.domain, True, ngrow=1, _post_barrier=False))
if rank == 0:
    for k, v in res.items(): print(f"world={world} {k:34s} {v:8.1f} us")
dist.barrier(device_ids=[local])
