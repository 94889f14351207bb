"""torchrun: do host<->device copies on side streams slow the distributed
MLMG's device barriers / fills / sweeps?  Per-op graph timings (as in
tools/mb_dist.py) with and without background pinned-memory copies."""
import os, sys, numpy as np, torch, torch.distributed as dist
sys.path.insert(0, '/root/repo')
world = int(os.environ.get("WORLD_SIZE", "1")); rank = int(os.environ.get("RANK", "0")); local = int(os.environ.get("LOCAL_RANK", "0"))
torch.cuda.set_device(local)
dist.init_process_group("nccl", device_id=torch.device("cuda", local))
import paper_2009_12009_b200 as A
from paper_2009_12009_b200._native import lib
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
n = 256 ** 3
h_in = torch.empty(n, dtype=torch.float64).pin_memory()
h_out = torch.empty(n, dtype=torch.float64).pin_memory()
d_in = torch.empty(n, dtype=torch.float64, device="cuda")
d_out = torch.empty(n, dtype=torch.float64, device="cuda")
cs, ds = torch.cuda.Stream(), torch.cuda.Stream()
def background(k):
    for _ in range(k):
        with torch.cuda.stream(cs): d_in.copy_(h_in, non_blocking=True)
        with torch.cuda.stream(ds): h_out.copy_(d_out, non_blocking=True)
def graph_time(fn, reps, copies):
    fn(); torch.cuda.synchronize(); dist.barrier(device_ids=[local])
    g = torch.cuda.CUDAGraph(); s = torch.cuda.Stream(); s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s, capture_error_mode="relaxed"):
            for _ in range(reps): fn()
    torch.cuda.current_stream().wait_stream(s); torch.cuda.synchronize(); dist.barrier(device_ids=[local])
    ts = []
    for _ in range(5):
        dist.barrier(device_ids=[local]); torch.cuda.synchronize()
        if copies: background(copies)
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); g.replay(); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1) * 1e3 / reps)
    t = torch.tensor([np.median(ts)], device="cuda"); dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return t.item()
ops = {
    "peer_barrier": (lambda: tr.peer_barrier(), 200, 8),
    "fill L0 w2": (lambda: mg._fill(top, top.phi[top.cur], 2), 100, 8),
    "sweep L0 (no fill)": (lambda: A.stencil.gsrb_sweep(top.phi[0], top.phi[1], top.rhs, top.dh), 20, 8),
    "coarse tail": (lambda: mg._coarse_tail(), 50, 8),
}
L1 = mg.levels[1]
nrm = torch.zeros(1, dtype=torch.float64, device="cuda")
ops.update({
    "sweep L0 (+fill w2)": (lambda: mg._sweep(top), 20, 8),
    "resid_restrict L0": (lambda: mg._resid_restrict(0), 20, 8),
    "sweep+norm L0": (lambda: mg._sweep(top, norm=nrm), 20, 8),
    "sweep L1 (+fill w2)": (lambda: mg._sweep(L1), 50, 8),
    "resid_restrict L1": (lambda: mg._resid_restrict(1), 50, 8),
    "prolong_sweep L0": (lambda: mg._prolong_sweep(0) if top.fuse else mg._prolong(0), 20, 8),
    "prolong_sweep L1": (lambda: mg._prolong_sweep(1) if L1.fuse else mg._prolong(1), 50, 8),
    "allmax": (lambda: mg._allmax(nrm), 200, 8),
})
for l in range(mg.grid_from, mg.tail):
    ops[f"level_grid L{l} down"] = ((lambda l=l: mg._level_grid(l, False)), 50, 8)
    ops[f"level_grid L{l} up"] = ((lambda l=l: mg._level_grid(l, True)), 50, 8)
mg._prime()
ops["iteration"] = (lambda: mg._body(), 5, 8)
ops["store_host"] = (lambda: lib().amrb_store_host(A.stencil.C.c_void_p(mg.norm.data_ptr()), A.stencil.C.c_void_p(mg.norm_host.data_ptr()), 1, A.stencil.stream_ptr()), 200, 8)
for k, (fn, reps, cp) in ops.items():
    a = graph_time(fn, reps, 0)
    b = graph_time(fn, reps, cp)
    if rank == 0:
        print(f"world={world} {k:22s} quiet {a:9.1f} us   with copies {b:9.1f} us", flush=True)
dist.barrier(device_ids=[local])
