"""ncu target: the C3 fine-level fused prolongation sweep (PROL mode) next to
the plain sweep, 8 launches each, on the solver's own level-0 / level-1
layouts."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2009_12009_b200 as A  # noqa: E402
from paper_2009_12009_b200 import stencil as S  # noqa: E402

dom = A.Box((0, 0, 0), (255, 255, 255))
ba = A.BoxArray([dom]).max_size(64)
dm = A.DistributionMapping.single_rank(len(ba))
tr = A.Transport(1)
mg = A.MLMG(A.Geometry(dom, (0.0,) * 3, (1.0,) * 3, True), ba, dm, transport=tr)
top, nx = mg.levels[0], mg.levels[1]
a, b, c = top.phi[0], top.phi[1], nx.phi[0]
for f in (a, top.rhs, c):
    f.storage.normal_()
A.fill_boundary(a, tr, top.domain, True, ngrow=2)
A.fill_boundary(c, tr, nx.domain, True, ngrow=1)
for _ in range(8):
    S.gsrb_sweep_prolong(a, b, top.rhs, top.dh, c)
    S.gsrb_sweep(a, b, top.rhs, top.dh)
torch.cuda.synchronize()
