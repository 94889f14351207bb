import sys, numpy as np, torch
sys.path.insert(0, '/root/repo')
import paper_2009_12009_b200 as A
from paper_2009_12009_b200 import stencil as S
dom = A.Box((0,0,0),(255,255,255)); ba = A.BoxArray([dom]).max_size(64)
dm = A.DistributionMapping.single_rank(len(ba)); tr = A.Transport(1)
geom = A.Geometry(dom, (0.0,)*3, (1.0,)*3, True)
mg = A.MLMG(geom, ba, dm, transport=tr)
top = mg.levels[0]
for f in top.phi: f.storage.normal_()
top.rhs.storage.normal_()
mg._produced(top.phi[0], 0); mg._produced(top.phi[1], 0)
def graph_time(fn, reps=20):
    fn(); fn(); torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph(); s = torch.cuda.Stream(); s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            for _ in range(reps): fn()
    torch.cuda.current_stream().wait_stream(s); torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); g.replay(); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1) * 1e3 / reps)
    return np.median(ts)
def plain():
    a, b = top.phi[top.cur], top.phi[1 - top.cur]
    A.fill_boundary(a, tr, top.domain, True, ngrow=2)
    S.gsrb_sweep(a, b, top.rhs, top.dh)
    top.cur = 1 - top.cur
def plain_nofill():
    a, b = top.phi[top.cur], top.phi[1 - top.cur]
    S.gsrb_sweep(a, b, top.rhs, top.dh)
    top.cur = 1 - top.cur
print("push sweep (mg._sweep)   %.1f us" % graph_time(lambda: mg._sweep(top)), "push=", top.push)
print("fill + plain sweep       %.1f us" % graph_time(plain))
print("plain sweep (no fill)    %.1f us" % graph_time(plain_nofill))
def pro():
    mg._prolong(0)
print("prolong (push)           %.1f us" % graph_time(pro), "push=", top.push)
from paper_2009_12009_b200.interlevel import prolong_from
def pro_plain():
    prolong_from(top.phi[top.cur], mg.levels[1].phi[mg.levels[1].cur], (2, 2, 2), add=True)
def pro_fill():
    pro_plain(); A.fill_boundary(top.phi[top.cur], tr, top.domain, True, ngrow=2)
print("prolong (plain)          %.1f us" % graph_time(pro_plain))
print("prolong + fill w2        %.1f us" % graph_time(pro_fill))
