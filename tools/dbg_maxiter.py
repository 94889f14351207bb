import sys, numpy as np
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import paper_2009_12009_b200 as A
from oracle import mlmg_ref as R
from helpers import tboxes
n, m = 64, 32
dom = A.Box((0, 0, 0), (n - 1,) * 3)
ba = A.BoxArray([dom]).max_size(m)
dm = A.DistributionMapping.single_rank(len(ba))
geom = A.Geometry(dom, (0.0,) * 3, (1.0,) * 3, True)
rng = np.random.default_rng(21)
rhs = rng.standard_normal((n, n, n)); rhs -= rhs.mean()
for mi in (100, 3):
    ref = R.OracleMLMG(((0, 0, 0), (n - 1,) * 3), tboxes(ba)).solve(rhs, rtol=1e-10, max_iter=mi)
    b = A.MultiFab(ba, dm, 1, 0); b.load_valid_from(dom, rhs)
    for graph in (True, False):
        mg = A.MLMG(geom, ba, dm, transport=A.Transport(1), use_graph=graph)
        phi = A.MultiFab(ba, dm, 1, 1)
        mg.solve(phi, b, rtol=1e-10, max_iter=mi)
        print(mi, graph, "dev", mg.iterations, [f"{x:.4e}" for x in mg.history[:4]], "ref", ref["iterations"], [f"{x:.4e}" for x in ref["history"][:4]], flush=True)
