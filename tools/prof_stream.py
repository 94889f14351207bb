"""A few launches of one fused sweep on the C3 fine-level layout (one 256^3 box,
ghosts 2) for ncu: python tools/prof_stream.py [sweep|norm|prolong] [kernel]"""
import sys, os
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2009_12009_b200 as A  # noqa: E402
from paper_2009_12009_b200 import stencil as S  # noqa: E402
from paper_2009_12009_b200._native import set_option  # noqa: E402

op = sys.argv[1] if len(sys.argv) > 1 else "sweep"
set_option("sweep_kernel", int(sys.argv[2]) if len(sys.argv) > 2 else 0)
dom = A.Box((0, 0, 0), (255, 255, 255))
ba = A.BoxArray([dom])
dm = A.DistributionMapping.single_rank(1)
a, b = A.MultiFab(ba, dm, 1, 2), A.MultiFab(ba, dm, 1, 2)
rhs = A.MultiFab(ba, dm, 1, 1)
g = torch.Generator(device="cuda").manual_seed(3)
a.storage.copy_(torch.randn(a.storage.shape, generator=g, device="cuda", dtype=torch.float64))
rhs.storage.copy_(torch.randn(rhs.storage.shape, generator=g, device="cuda", dtype=torch.float64))
c = A.MultiFab(A.coarsened_layout(ba, 2), dm, 1, 1)
nrm = torch.zeros(1, dtype=torch.int64, device="cuda")
dh = (65536.0,) * 3
for _ in range(6):
    if op == "sweep":
        S.gsrb_sweep(a, b, rhs, dh)
    elif op == "norm":
        S.gsrb_sweep_norm(a, b, rhs, dh, nrm)
    else:
        S.gsrb_sweep_prolong(a, b, rhs, dh, c)
torch.cuda.synchronize()
print("ok", op)
