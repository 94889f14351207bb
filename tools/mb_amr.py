"""Device two-level advection step on the reference's own hierarchy
(tools/ref_amr_<n>.json): ms per coarse step, cell updates/s."""
import json, sys, time, numpy as np, torch
sys.path.insert(0, '/root/repo')
import paper_2009_12009_b200 as A
from paper_2009_12009_b200 import amr
for fn in sys.argv[1:]:
    d = json.load(open(fn)); n = d["n"]; dim = 3
    dom = A.Box((0, 0, 0), (n - 1,) * 3)
    geom = A.Geometry(dom, (0.0,) * 3, (1.0,) * 3, (True,) * 3)
    mk = lambda rows: A.BoxArray([A.Box(r[:3], r[3:]) for r in rows])
    ba0, ba1 = mk(d["ba0"]), mk(d["ba1"])
    s = amr.AdvectionSolver(geom, ba0, A.DistributionMapping.single_rank(len(ba0)), ba1,
                            A.DistributionMapping.single_rank(len(ba1)), (2, 2, 2), (1.0, 0.5, 0.25), cfl=0.4)
    for lev in (0, 1):
        s.phi[lev].storage.normal_()
    for _ in range(3):
        s.step()
    torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        t0 = time.perf_counter(); s.step(); torch.cuda.synchronize(); ts.append(time.perf_counter() - t0)
    t = min(ts)
    upd = d["coarse_cells"] + 2 * d["fine_cells"]
    print(f"n={n}: {len(ba0)} coarse boxes, {len(ba1)} fine boxes; device step {t*1e3:.2f} ms "
          f"({upd/t/1e6:.1f} M cell-updates/s); reference CPU step {d['step_s']*1e3:.0f} ms -> x{d['step_s']/t:.0f}")
