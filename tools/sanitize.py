"""Small invocations of the concurrency-heavy kernels, for the checked build
(device invariant checks; compute-sanitizer is closed on this GPU pool):

    AMRB_LIBRARY=checked python tools/sanitize.py

* k_gsrb_stream: plain, NORM, PROL, with and without the ghost push, one box
  and a multi-box layout (TMA ring + mbarriers + fence.proxy.async, one
  __syncthreads per step, two directions);
* the MLMG coarse tail on an 8-CTA cluster (DSMEM) and the one-CTA tail;
* k_level_grid (cooperative grid.sync);
* k_copy fills (FillBoundary copy programs);
* the device solve loop (WHILE-node graph) of a small MLMG.
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2009_12009_b200 as A  # noqa: E402
from paper_2009_12009_b200 import stencil as S  # noqa: E402
from paper_2009_12009_b200.ghosts import push_table  # noqa: E402

torch.cuda.set_device(0)
rng = np.random.default_rng(5)
DH = (4096.0,) * 3
for n, m in ((64, 64), (64, 32), (128, 64)):
    dom = A.Box((0, 0, 0), (n - 1,) * 3)
    ba = A.BoxArray([dom]).max_size(m)
    dm = A.DistributionMapping.single_rank(len(ba))
    tr = A.Transport(1)
    a, b, rhs = A.MultiFab(ba, dm, 1, 2), A.MultiFab(ba, dm, 1, 2), A.MultiFab(ba, dm, 1, 1)
    a.load_valid_from(dom, rng.normal(size=(n, n, n)))
    rhs.load_valid_from(dom, rng.normal(size=(n, n, n)))
    A.fill_boundary(a, tr, dom, True)
    A.fill_boundary(rhs, tr, dom, True)
    c = A.MultiFab(A.coarsened_layout(ba, 2), dm, 1, 1)
    A.fill_boundary(c, tr, dom.coarsen(2), True)
    nrm = torch.zeros(1, dtype=torch.int64, device="cuda")
    tab = push_table(b, dom, True, 2)
    for push in (None, tab):
        S.gsrb_sweep(a, b, rhs, DH, push=push)
        S.gsrb_sweep_norm(a, b, rhs, DH, nrm, push=push)
        S.gsrb_sweep_prolong(a, b, rhs, DH, c, push=push)
    torch.cuda.synchronize()
    print("stream kernels ok", n, m, flush=True)
for n, m, ct in ((64, 32, 1), (32, 16, 0), (128, 64, 1)):
    dom = A.Box((0, 0, 0), (n - 1,) * 3)
    ba = A.BoxArray([dom]).max_size(m)
    dm = A.DistributionMapping.single_rank(len(ba))
    geom = A.Geometry(dom, (0.0,) * 3, (1.0,) * 3, True)
    g = rng.normal(size=(n, n, n))
    g -= g.mean()
    rhs = A.MultiFab(ba, dm, 1, 0)
    rhs.load_valid_from(dom, g)
    phi = A.MultiFab(ba, dm, 1, 1)
    mg = A.MLMG(geom, ba, dm, cluster_tail=ct)
    mg.solve(phi, rhs, rtol=1e-10, max_iter=4)
    torch.cuda.synchronize()
    print("mlmg ok", n, m, "cluster", mg.cluster_tail, "grid levels", mg.tail - mg.grid_from, flush=True)
from paper_2009_12009_b200._native import LIB_PATH, debug_checks  # noqa: E402

fails, line = debug_checks()
print(f"library {os.path.basename(LIB_PATH)}: DCHECK failures {fails} (first at line {line})", flush=True)
print("SANITIZE_DRIVER_DONE", flush=True)
