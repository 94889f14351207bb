import sys, numpy as np, torch
sys.path.insert(0, '/root/repo')
import paper_2009_12009_b200 as A
from paper_2009_12009_b200 import stencil as S
from paper_2009_12009_b200._native import option
from paper_2009_12009_b200.ghosts import pull_table
DH = (65536.0, 16384.0, 4096.0)
rng = np.random.default_rng(0)
n = m = 64
dom = A.Box([0] * 3, [n - 1] * 3)
ba = A.BoxArray([dom]).max_size(m)
dm = A.DistributionMapping.single_rank(len(ba))
tr = A.Transport(1); p3 = (True,) * 3
g = rng.normal(size=(1, n, n, n)); gr = rng.normal(size=(1, n, n, n))
a = A.MultiFab(ba, dm, 1, 2); a.load_valid_from(dom, g); A.fill_boundary(a, tr, dom, p3)
rhs = A.MultiFab(ba, dm, 1, 1); rhs.load_valid_from(dom, gr); A.fill_boundary(rhs, tr, dom, p3)
for segs in (1, 2, 4, 0):
  for alt in (0, 1):
    a2 = A.MultiFab(ba, dm, 1, 2); a2.setval(-7777.0); a2.load_valid_from(dom, g)
    tab = pull_table(a2, dom, p3, 2)
    b2 = A.MultiFab(ba, dm, 1, 2)
    with option("stream_segments", segs), option("stream_alternate", alt):
        S.gsrb_sweep_pull(a2, b2, rhs, DH, tab)
    torch.cuda.synchronize()
    x = a.fab(0).data.cpu().numpy()[0]; y = a2.fab(0).data.cpu().numpy()[0]
    bad = np.argwhere(x != y) - 2
    cls = {}
    for b in bad:
        d = tuple(-1 if c < 0 else (1 if c >= n else 0) for c in b)
        cls[d] = cls.get(d, 0) + 1
    print("segs", segs, "alt", alt, "missing", len(bad), sorted(cls.items())[:12], flush=True)
