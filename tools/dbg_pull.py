import sys, numpy as np, torch
sys.path.insert(0, '/root/repo')
import paper_2009_12009_b200 as A
from paper_2009_12009_b200 import stencil as S
from paper_2009_12009_b200.ghosts import pull_table
DH = (65536.0, 16384.0, 4096.0)
rng = np.random.default_rng(0)
for n, m in [(64, 64), (64, 32), (128, 64)]:
    dom = A.Box([0] * 3, [n - 1] * 3)
    ba = A.BoxArray([dom]).max_size(m)
    dm = A.DistributionMapping.single_rank(len(ba))
    tr = A.Transport(1)
    p3 = (True,) * 3
    g = rng.normal(size=(1, n, n, n)); gr = rng.normal(size=(1, n, n, n))
    a = A.MultiFab(ba, dm, 1, 2); a.load_valid_from(dom, g); A.fill_boundary(a, tr, dom, p3)
    rhs = A.MultiFab(ba, dm, 1, 1); rhs.load_valid_from(dom, gr); A.fill_boundary(rhs, tr, dom, p3)
    ref = A.MultiFab(ba, dm, 1, 2); S.gsrb_sweep(a, ref, rhs, DH)
    a2 = A.MultiFab(ba, dm, 1, 2); a2.setval(-7777.0); a2.load_valid_from(dom, g)
    tab = pull_table(a2, dom, p3, 2)
    print(n, m, "table", None if tab is None else tab.host.shape, flush=True)
    b2 = A.MultiFab(ba, dm, 1, 2)
    S.gsrb_sweep_pull(a2, b2, rhs, DH, tab)
    torch.cuda.synchronize()
    for i in a.fabs:
        x = a.fab(i).data.cpu().numpy()[0]; y = a2.fab(i).data.cpu().numpy()[0]
        bad = np.argwhere(x != y)
        if len(bad):
            print(" box", i, "ghost mismatches", len(bad), "first", bad[:5].tolist(), "vals", [y[tuple(b)] for b in bad[:3]], [x[tuple(b)] for b in bad[:3]])
            # per-face summary
            print("   i-range", bad[:,0].min(), bad[:,0].max(), "j", bad[:,1].min(), bad[:,1].max(), "k", bad[:,2].min(), bad[:,2].max())
        u = ref.fab(i).valid().cpu().numpy(); v = b2.fab(i).valid().cpu().numpy()
        print(" box", i, "out mismatches", int((u != v).sum()))
    d = tab.host.reshape(-1, 27)[0]
    base = a2.storage.data_ptr()
    print(" tab box0 (offsets rel. storage, elements):", [((int(x) & ~1) - base) // 8 if x else 0 for x in d])
    print(" fabtab0", a2.fabtab[0].tolist(), "ngrow", a2.ngrow)
