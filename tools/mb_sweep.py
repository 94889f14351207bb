import sys, numpy as np, torch, json
sys.path.insert(0, '/root/repo')
import paper_2009_12009_b200 as A
from paper_2009_12009_b200 import stencil as S
res = {}
import os
cfgs = [tuple(int(x) for x in c.split('/')) for c in os.environ.get('MB_CFGS', '256/64,256/256,128/32,512/32').split(',')]
for n, m in cfgs:
    dom = A.Box((0,0,0),(n-1,)*3); ba = A.BoxArray([dom]).max_size(m)
    dm = A.DistributionMapping.single_rank(len(ba)); tr = A.Transport(1)
    a = A.MultiFab(ba, dm, 1, 2); b = A.MultiFab(ba, dm, 1, 2); r = A.MultiFab(ba, dm, 1, 1)
    a.storage.normal_(); r.storage.normal_()
    dh = (float(n*n),)*3
    ts = []; tf = []
    for it in range(25):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True); e2 = torch.cuda.Event(enable_timing=True)
        e0.record()
        A.fill_boundary(a, tr, dom, True)
        e1.record()
        S.gsrb_sweep(a, b, r, dh)
        e2.record()
        a, b = b, a
        ts.append((e1, e2)); tf.append((e0, e1))
    torch.cuda.synchronize()
    t = np.median([x.elapsed_time(y) for x, y in ts[5:]]) * 1e3
    f = np.median([x.elapsed_time(y) for x, y in tf[5:]]) * 1e3
    N = n**3; F = len(ba) * 6 * m * m
    gbs = (24 * N + 8 * F) / t / 1e3
    print(f"{n}^3/{m}^3: sweep {t:8.1f} us  {gbs:7.1f} GB/s  {gbs/6534.5*100:5.1f}%   fill(w2) {f:7.1f} us   {N/t/1e3:.1f} G upd/s")
