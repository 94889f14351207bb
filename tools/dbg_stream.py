import numpy as np, torch, sys
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import paper_2009_12009_b200 as A
from paper_2009_12009_b200 import stencil as S
from paper_2009_12009_b200._native import option
rng = np.random.default_rng(0)
n=64
dom = A.Box((0,0,0),(n-1,)*3); ba = A.BoxArray([dom]).max_size(64); dm = A.DistributionMapping.single_rank(1)
tr = A.Transport(1)
a = A.MultiFab(ba, dm, 1, 2); rhs = A.MultiFab(ba, dm, 1, 1)
a.load_valid_from(dom, rng.normal(size=(1,n,n,n))); rhs.load_valid_from(dom, rng.normal(size=(1,n,n,n)))
A.fill_boundary(a, tr, dom, True); A.fill_boundary(rhs, tr, dom, True)
DH=(65536.0, 16384.0, 4096.0)
out={}
for k in (0,1):
    b = A.MultiFab(ba, dm, 1, 2)
    with option("sweep_kernel", k):
        S.gsrb_sweep(a, b, rhs, DH)
    torch.cuda.synchronize()
    out[k] = b.fab(0).valid().cpu().numpy()[0]
d = out[0] != out[1]
print("mismatches", d.sum(), "of", d.size)
idx = np.argwhere(d)
print(idx[:40])
for ax in range(3):
    print("axis", ax, np.bincount(idx[:,ax], minlength=n))
par = (idx.sum(1)) % 2
print("parity counts (0=red)", np.bincount(par))
for opt in (("stream_segments", 1), ("stream_alternate", 0)):
    with option(*opt):
        b = A.MultiFab(ba, dm, 1, 2)
        S.gsrb_sweep(a, b, rhs, DH)
        torch.cuda.synchronize()
        d = b.fab(0).valid().cpu().numpy()[0] != out[1]
        print(opt, "mismatches", d.sum(), "planes", np.nonzero(d.any(axis=(1, 2)))[0][:20])
