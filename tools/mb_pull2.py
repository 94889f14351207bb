"""Which part of the in-kernel ghost pull costs: time the pull sweep with the
table restricted to subsets of directions (1 GPU, 256^3 single box)."""
import sys, itertools, numpy as np, torch
sys.path.insert(0, '/root/repo')
import paper_2009_12009_b200 as A
from paper_2009_12009_b200 import stencil as S
from paper_2009_12009_b200.ghosts import pull_table, PushTable
exec(open('/root/repo/tools/mb_pull.py').read().split("prof = ")[0].split("rng = np.random.default_rng(0)")[1])
DH = (65536.0, 16384.0, 4096.0)
n = m = int(sys.argv[1]) if len(sys.argv) > 1 else 256
dom = A.Box([0] * 3, [n - 1] * 3)
ba = A.BoxArray([dom]).max_size(m)
dm = A.DistributionMapping.single_rank(len(ba))
tr = A.Transport(1); p3 = (True,) * 3
a = A.MultiFab(ba, dm, 1, 2); a.storage.normal_(); A.fill_boundary(a, tr, dom, p3)
rhs = A.MultiFab(ba, dm, 1, 1); rhs.storage.normal_(); A.fill_boundary(rhs, tr, dom, p3)
b = A.MultiFab(ba, dm, 1, 2)
full = pull_table(a, dom, p3, 2)
dirs = [d for d in itertools.product((-1, 0, 1), repeat=3)]
def sub(pred):
    h = full.host.copy().reshape(-1, 27)
    for x, d in enumerate(dirs):
        if not pred(d): h[:, x] = 0
    return PushTable(h, False, 2, a.device)
cases = {"none": sub(lambda d: False), "i only": sub(lambda d: d[0] != 0 and d[1] == 0 and d[2] == 0),
         "j only": sub(lambda d: d[1] != 0 and d[0] == 0 and d[2] == 0), "k only": sub(lambda d: d[2] != 0 and d[0] == 0 and d[1] == 0),
         "all": full}
print(f"{n}^3/{m} plain sweep {gt(lambda: S.gsrb_sweep(a, b, rhs, DH)):7.1f} us", flush=True)
for k, t in cases.items():
    print(f"  pull {k:8s} {gt(lambda: S.gsrb_sweep_pull(a, b, rhs, DH, t)):7.1f} us", flush=True)
