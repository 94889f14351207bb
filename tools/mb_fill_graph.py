import sys, numpy as np, torch
sys.path.insert(0, '/root/repo')
import paper_2009_12009_b200 as A
from paper_2009_12009_b200 import stencil as S
for n, m, g in ((256, 256, 2), (256, 256, 1), (256, 64, 2), (512, 32, 1)):
    dom = A.Box((0,0,0),(n-1,)*3); ba = A.BoxArray([dom]).max_size(m)
    dm = A.DistributionMapping.single_rank(len(ba)); tr = A.Transport(1)
    a = A.MultiFab(ba, dm, 1, 2); a.storage.normal_()
    b = A.MultiFab(ba, dm, 1, 2); r = A.MultiFab(ba, dm, 1, 1); r.storage.normal_()
    dh = (float(n*n),)*3
    A.fill_boundary(a, tr, dom, True, ngrow=g); S.gsrb_sweep(a, b, r, dh); torch.cuda.synchronize()
    s = torch.cuda.Stream()
    for what in ("fill", "sweep", "fill+sweep"):
        gr = torch.cuda.CUDAGraph()
        with torch.cuda.stream(s):
            with torch.cuda.graph(gr, stream=s):
                for _ in range(20):
                    if "fill" in what: A.fill_boundary(a, tr, dom, True, ngrow=g)
                    if "sweep" in what: S.gsrb_sweep(a, b, r, dh)
        torch.cuda.synchronize()
        ts = []
        for _ in range(5):
            e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
            e0.record(); gr.replay(); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1) * 1e3 / 20)
        print(f"{n}^3/{m}^3 g={g} {what:11s} {np.median(ts):8.1f} us (graph, warm)")
