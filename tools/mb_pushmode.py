import sys, numpy as np, torch
sys.path.insert(0, '/root/repo')
import paper_2009_12009_b200 as A
dom = A.Box((0,0,0),(255,255,255)); ba = A.BoxArray([dom]).max_size(64)
dm = A.DistributionMapping.single_rank(len(ba))
geom = A.Geometry(dom, (0.0,)*3, (1.0,)*3, True)
rhs = A.MultiFab(ba, dm, 1, 0)
for f in rhs.fabs.values(): f.valid().normal_()
mu = sum(float(f.valid().sum()) for f in rhs.fabs.values()) / ba.num_cells()
for f in rhs.fabs.values(): f.valid().sub_(mu)
for mode in (False, "coarse", True):
    mg = A.MLMG(geom, ba, dm, transport=A.Transport(1), ghost_push=mode)
    phi = A.MultiFab(ba, dm, 1, 1)
    mg.solve(phi, rhs); torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        phi.setval(0.0); torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); mg.solve(phi, rhs); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
    print(f"ghost_push={mode!s:7s} solve {np.median(ts):.3f} ms iters {mg.iterations} push levels {[l for l, lv in enumerate(mg.levels) if lv.push]}")
