"""Graph timings: plain sweep, fill + sweep, in-kernel pull sweep (1 GPU)."""
import sys, numpy as np, torch
sys.path.insert(0, '/root/repo')
import paper_2009_12009_b200 as A
from paper_2009_12009_b200 import stencil as S
from paper_2009_12009_b200.ghosts import pull_table
DH = (65536.0, 16384.0, 4096.0)
rng = np.random.default_rng(0)
def gt(fn, reps=20):
    fn(); torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph(); s = torch.cuda.Stream(); s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            for _ in range(reps): fn()
    torch.cuda.current_stream().wait_stream(s); torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); g.replay(); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1) * 1e3 / reps)
    return float(np.median(ts))
prof = len(sys.argv) > 1
for n, m in ([(256, 256)] if prof else [(256, 256), (128, 128), (256, 64)]):
    dom = A.Box([0] * 3, [n - 1] * 3)
    ba = A.BoxArray([dom]).max_size(m)
    dm = A.DistributionMapping.single_rank(len(ba))
    tr = A.Transport(1); p3 = (True,) * 3
    a = A.MultiFab(ba, dm, 1, 2); a.storage.normal_(); A.fill_boundary(a, tr, dom, p3)
    rhs = A.MultiFab(ba, dm, 1, 1); rhs.storage.normal_(); A.fill_boundary(rhs, tr, dom, p3)
    b = A.MultiFab(ba, dm, 1, 2)
    tab = pull_table(a, dom, p3, 2)
    if prof:
        for _ in range(3): S.gsrb_sweep_pull(a, b, rhs, DH, tab)
        torch.cuda.synchronize(); break
    t0 = gt(lambda: S.gsrb_sweep(a, b, rhs, DH))
    t1 = gt(lambda: (A.fill_boundary(a, tr, dom, p3, ngrow=2), S.gsrb_sweep(a, b, rhs, DH)))
    t2 = gt(lambda: S.gsrb_sweep_pull(a, b, rhs, DH, tab))
    print(f"{n}^3/{m}: sweep {t0:7.1f} us   fill+sweep {t1:7.1f} us   pull sweep {t2:7.1f} us", flush=True)
