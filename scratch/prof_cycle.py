import sys, numpy as np, torch, collections
sys.path.insert(0, '/root/repo')
import paper_2009_12009_b200 as A
from paper_2009_12009_b200 import mlmg as MM
n, m = 256, 64
dom = A.Box((0,0,0),(n-1,)*3); ba = A.BoxArray([dom]).max_size(m)
dm = A.DistributionMapping.single_rank(len(ba)); geom = A.Geometry(dom,(0.,)*3,(1.,)*3,True)
rhs = A.MultiFab(ba, dm, 1, 0); rhs.storage.normal_()
phi = A.MultiFab(ba, dm, 1, 1)
mg = A.MLMG(geom, ba, dm, use_graph=False)
mg.solve(phi, rhs, rtol=1e-3, max_iter=2)
rec = []
def wrap(name, fn):
    def w(*a, **k):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); r = fn(*a, **k); e1.record()
        lvl = None
        if a and hasattr(a[0], 'domain'): lvl = a[0].domain.extents()[0]
        elif a and isinstance(a[0], int): lvl = mg.levels[a[0]].domain.extents()[0]
        rec.append((name, lvl, e0, e1)); return r
    return w
orig = {}
for nm in ('_fill', '_sweep', '_resid_restrict', '_prolong', '_coarse_tail', '_residual_norm'):
    orig[nm] = getattr(mg, nm)
    setattr(mg, nm, wrap(nm, orig[nm]))
# _fill inside _sweep/_resid is counted separately; compute exclusive later
torch.cuda.synchronize()
for _ in range(3):
    rec.clear()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(); mg._cycle_and_norm(); e1.record(); torch.cuda.synchronize()
tot = e0.elapsed_time(e1)*1e3
agg = collections.defaultdict(float); cnt = collections.Counter()
for name, lvl, a, b in rec:
    agg[(name, lvl)] += a.elapsed_time(b)*1e3; cnt[(name, lvl)] += 1
print(f"cycle+norm: {tot:.1f} us")
for k in sorted(agg, key=lambda k: -agg[k]):
    print(f"{k[0]:16s} lvl {str(k[1]):5s} x{cnt[k]:3d}  {agg[k]:9.1f} us")
