"""Reference AdvectionSolver timing (CPU, this container) + hierarchy dump for
the device benchmark (tools/mb_amr.py)."""
import json, sys, time
sys.path.insert(0, "/root/reference/pkg/src")
import numpy as np
import amrkit
from amrkit.advect import AdvectionSolver
from amrkit.amr_core import Geometry, GridGenParams
dim, n, mg, bf = 3, int(sys.argv[1]) if len(sys.argv) > 1 else 64, 16, 8
dom = amrkit.Box(amrkit.IntVect.zero(dim), amrkit.IntVect([n - 1] * dim))
geom = Geometry(dom, (0.0,) * dim, (1.0,) * dim, (True,) * dim)
params = GridGenParams(dim=dim, max_level=1, max_grid_size=mg, blocking_factor=bf)
t0 = time.perf_counter()
s = AdvectionSolver(geom, params, velocity=(1.0, 0.5, 0.25), nranks=1, cfl=0.4, use_reflux=True)
t1 = time.perf_counter()
ts = []
for _ in range(2):
    a = time.perf_counter(); s.step(); ts.append(time.perf_counter() - a)
ncf = sum(b.num_cells() for b in s.hier.ba(1))
print(json.dumps({"n": n, "setup_s": t1 - t0, "step_s": min(ts), "coarse_cells": n ** 3, "fine_cells": ncf,
                  "ba0": [list(b.lo) + list(b.hi) for b in s.hier.ba(0)],
                  "ba1": [list(b.lo) + list(b.hi) for b in s.hier.ba(1)]}))
