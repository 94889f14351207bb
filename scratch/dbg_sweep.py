import sys, numpy as np, torch
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import paper_2009_12009_b200 as A
from paper_2009_12009_b200 import stencil as S
from oracle import mlmg_ref as R, mesh_ref as M
from helpers import tboxes
DH=(1.0,1.0,1.0)
for n, m in ((8,8),(16,8),(16,16)):
    dom = A.Box((0,0,0),(n-1,)*3); ba = A.BoxArray([dom]).max_size(m)
    dm = A.DistributionMapping.single_rank(len(ba)); tr=A.Transport(1)
    rng=np.random.default_rng(0)
    g=rng.standard_normal((1,n,n,n)); gr=rng.standard_normal((1,n,n,n))
    a=A.MultiFab(ba,dm,1,2); b=A.MultiFab(ba,dm,1,2); rhs=A.MultiFab(ba,dm,1,1)
    a.load_valid_from(dom,g); rhs.load_valid_from(dom,gr); A.fill_boundary(rhs,tr,dom,True)
    A.fill_boundary(a,tr,dom,True); S.gsrb_sweep(a,b,rhs,DH)
    boxes=tboxes(ba); d=((0,0,0),(n-1,)*3)
    pf=M.make_fabs(boxes,1,1); rf=M.make_fabs(boxes,1,0)
    M.load_global(boxes,pf,1,d,g); M.load_global(boxes,rf,0,d,gr)
    M.fill_boundary(boxes,pf,1,d,(True,)*3)
    for i,bx in enumerate(boxes): R.gsrb_color(bx,pf[i][0],rf[i][0],DH,0)
    red = M.gather(boxes,pf,1,d)
    M.fill_boundary(boxes,pf,1,d,(True,)*3)
    for i,bx in enumerate(boxes): R.gsrb_color(bx,pf[i][0],rf[i][0],DH,1)
    want = M.gather(boxes,pf,1,d)
    have = A.gather_global(b, dom)
    bad = np.argwhere(have != want)
    par = (bad.sum(axis=1)) % 2
    print(n, m, "bad cells", len(bad), "of", n**3, "red-bad", (par==0).sum(), "black-bad", (par==1).sum())
    redbad = np.argwhere((have != red) & ((np.indices((n,)*3).sum(0)%2)==0))
    print("  red cells != oracle red:", len(redbad), redbad[:10].tolist())
    print("  sample bad:", bad[:20].tolist())
