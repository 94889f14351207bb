import sys, numpy as np, torch
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import paper_2009_12009_b200 as A
from oracle import mlmg_ref as R, mesh_ref as M
from helpers import tboxes
n, m = 32, 16
dom = A.Box((0,0,0),(n-1,)*3); ba = A.BoxArray([dom]).max_size(m)
dm = A.DistributionMapping.single_rank(len(ba)); geom = A.Geometry(dom,(0.,)*3,(1.,)*3,True)
rng = np.random.default_rng(1); rhs = rng.standard_normal((n,n,n)); rhs -= rhs.mean()
mg = A.MLMG(geom, ba, dm, use_graph=False)
o = R.OracleMLMG(((0,0,0),(n-1,)*3), tboxes(ba))
b = A.MultiFab(ba, dm, 1, 0); b.load_valid_from(dom, rhs)
phi = A.MultiFab(ba, dm, 1, 1)
mg.set_rhs(b); mg.set_phi(phi)
top = o.levels[0]
M.load_global(top['boxes'], top['rhs'], 0, top['domain'], rhs[None])
def cmp(l, what):
    lv = mg.levels[l]; olv = o.levels[l]
    if what == 'phi':
        d = lv.phi[lv.cur]; of = olv['phi']; ng = 1; dng = 2
    else:
        d = lv.rhs; of = olv['rhs']; ng = 0; dng = 1
    worst = 0
    for i, f in d.fabs.items():
        have = f.valid().cpu().numpy()
        want = M.valid(olv['boxes'], of, ng, i)
        worst = max(worst, np.abs(have-want).max())
    print(f"level {l} {what}: max|diff| = {worst:.3e}")
L = len(mg.levels)
print([ (lv.kind, len(lv.ba), lv.domain) for lv in mg.levels])
for l in range(L-1):
    if l > 0:
        mg.levels[l].phi[mg.levels[l].cur].storage.zero_()
        for f in o.levels[l]['phi'].values(): f[...] = 0
    mg._smooth(mg.levels[l], 2); o.smooth(o.levels[l], 2); torch.cuda.synchronize(); cmp(l, 'phi')
    mg._resid_restrict(l)
    r = o.residual(o.levels[l]); M.average_down(o.levels[l]['boxes'], r, 0, o.levels[l+1]['boxes'], o.levels[l+1]['rhs'], 0, (2,2,2))
    torch.cuda.synchronize(); cmp(l+1, 'rhs')
bot = mg.levels[-1]; bot.phi[bot.cur].storage.zero_()
for f in o.levels[-1]['phi'].values(): f[...] = 0
mg._smooth(bot, 32); o.smooth(o.levels[-1], 32); torch.cuda.synchronize(); cmp(L-1, 'phi')
for l in range(L-2, -1, -1):
    mg._prolong(l); M.interp_pc(o.levels[l]['boxes'], o.levels[l]['phi'], 1, o.levels[l+1]['boxes'], o.levels[l+1]['phi'], 1, (2,2,2), add=True)
    torch.cuda.synchronize(); cmp(l, 'phi')
    mg._smooth(mg.levels[l], 2); o.smooth(o.levels[l], 2); torch.cuda.synchronize(); cmp(l, 'phi')
