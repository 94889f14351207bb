import sys, torch, numpy as np
sys.path.insert(0, '/root/repo')
import paper_2009_12009_b200 as A
from paper_2009_12009_b200 import stencil as S
n, m = 256, 64
dom = A.Box((0,0,0),(n-1,)*3); ba = A.BoxArray([dom]).max_size(m)
dm = A.DistributionMapping.single_rank(len(ba)); tr = A.Transport(1)
a = A.MultiFab(ba, dm, 1, 2); b = A.MultiFab(ba, dm, 1, 2); r = A.MultiFab(ba, dm, 1, 1); o = A.MultiFab(ba, dm, 1, 0)
a.storage.normal_(); r.storage.normal_()
def t(fn, nb, name):
    for _ in range(3): fn()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20): fn()
    e1.record(); torch.cuda.synchronize()
    us = e0.elapsed_time(e1)/20*1e3
    print(f"{name:50s} {us:8.1f} us  {nb/us/1e3:7.0f} GB/s")
N = n**3
t(lambda: torch.add(a.storage[:r.storage.numel()], r.storage, out=b.storage[:r.storage.numel()]), 3*r.storage.numel()*8, "torch add on multifab storages (contig)")
t(lambda: S.residual(o, r, a, (1.,1.,1.)), 3*N*8, "k_stencil residual (3 streams valid)")
t(lambda: S.laplacian(o, a, (1.,1.,1.)), 2*N*8, "k_stencil lap (2 streams)")
dh=(float(n*n),)*3
t(lambda: S.gsrb_sweep(a, b, r, dh), 24*N, "gsrb_sweep")
