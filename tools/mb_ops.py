import sys, numpy as np, torch
sys.path.insert(0, '/root/repo')
import paper_2009_12009_b200 as A
dom = A.Box((0,0,0),(255,255,255)); ba = A.BoxArray([dom]).max_size(64)
dm = A.DistributionMapping.single_rank(len(ba)); tr = A.Transport(1)
geom = A.Geometry(dom, (0.0,)*3, (1.0,)*3, True)
mg = A.MLMG(geom, ba, dm, transport=tr)
for lv in mg.levels:
    for f in lv.phi: f.storage.normal_()
    lv.rhs.storage.normal_()
def tm(fn, n=20):
    ev = []
    for _ in range(n):
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); ev.append((a, b))
    torch.cuda.synchronize()
    return np.median([x.elapsed_time(y) for x, y in ev[3:]]) * 1e3
top = mg.levels[0]
res = {}
res['fill w1'] = tm(lambda: mg._fill(top, top.phi[top.cur], 1))
res['fill w2'] = tm(lambda: mg._fill(top, top.phi[top.cur], 2))
res['sweep (incl fill w2)'] = tm(lambda: mg._sweep(top))
res['resid_restrict (incl fill w1)'] = tm(lambda: mg._resid_restrict(0))
res['prolong'] = tm(lambda: mg._prolong(0))
res['residual_norm (incl fill w1)'] = tm(lambda: mg._residual_norm())
res['vcycle+norm'] = tm(lambda: mg._cycle_and_norm(), 10)
for k, v in res.items(): print(f"{k:32s} {v:9.1f} us")
