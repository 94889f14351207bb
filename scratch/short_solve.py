import sys, torch
sys.path.insert(0, '/root/repo')
import paper_2009_12009_b200 as A
n, m = 256, 64
dom = A.Box((0,0,0),(n-1,)*3); ba = A.BoxArray([dom]).max_size(m)
dm = A.DistributionMapping.single_rank(len(ba)); geom = A.Geometry(dom,(0.,)*3,(1.,)*3,True)
rhs = A.MultiFab(ba, dm, 1, 0); rhs.storage.normal_()
phi = A.MultiFab(ba, dm, 1, 1)
mg = A.MLMG(geom, ba, dm)
mg.solve(phi, rhs, rtol=1e-30, max_iter=3)
torch.cuda.synchronize()
print("ok", mg.iterations)
