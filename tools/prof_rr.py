import sys, torch
sys.path.insert(0, '/root/repo')
import paper_2009_12009_b200 as A
dom = A.Box((0,0,0),(255,255,255)); ba = A.BoxArray([dom]).max_size(64)
dm = A.DistributionMapping.single_rank(len(ba)); tr = A.Transport(1)
geom = A.Geometry(dom, (0.0,)*3, (1.0,)*3, True)
mg = A.MLMG(geom, ba, dm, transport=tr)
for lv in mg.levels:
    for f in lv.phi: f.storage.normal_()
    lv.rhs.storage.normal_()
for _ in range(6):
    mg._resid_restrict(0); mg._residual_norm()
torch.cuda.synchronize()
