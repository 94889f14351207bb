"""Graph-replayed fill + sweep on the C3 solver's level-1 and level-2 layouts
(one 128^3 / 64^3 box), for tile-variant A/B runs (AMRB_SWEEP_IMPL / _TK)."""
import sys, numpy as np, torch
sys.path.insert(0, '/root/repo')
import paper_2009_12009_b200 as A
from paper_2009_12009_b200 import stencil as S
for n in (128, 64):
    dom = A.Box((0,0,0),(n-1,)*3); ba = A.BoxArray([dom])
    dm = A.DistributionMapping.single_rank(1); tr = A.Transport(1)
    a = A.MultiFab(ba, dm, 1, 2); b = A.MultiFab(ba, dm, 1, 2); r = A.MultiFab(ba, dm, 1, 1)
    a.storage.normal_(); r.storage.normal_(); dh = (float(n*n),)*3
    def both():
        A.fill_boundary(a, tr, dom, True, ngrow=2); S.gsrb_sweep(a, b, r, dh)
    def sweep():
        S.gsrb_sweep(a, b, r, dh)
    for name, fn in (("fill+sweep", both), ("sweep", sweep)):
        fn(); torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph(); s = torch.cuda.Stream(); s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            with torch.cuda.graph(g, stream=s):
                for _ in range(20): fn()
        torch.cuda.synchronize(); ts = []
        for _ in range(5):
            e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
            e0.record(); g.replay(); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1) * 1e3 / 20)
        print(f"  {n}^3 {name:10s} {np.median(ts):7.2f} us")
