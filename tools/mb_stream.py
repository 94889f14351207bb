"""Microbenchmark: fused GSRB sweep kernels, k_gsrb_stream vs the previous TMA
kernels (library option sweep_kernel = 0 / 1), CUDA events on the launch
stream, warm, averaged; plus the NORM and PROL variants.

    python tools/mb_stream.py [--reps 20]
"""

import argparse
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2009_12009_b200 as A  # noqa: E402
from paper_2009_12009_b200 import stencil as S  # noqa: E402
from paper_2009_12009_b200._native import option  # noqa: E402

PEAK = 6552.0
CONFIGS = [int(x) for x in os.environ.get("MB_CONFIGS", "0,1,2,4").split(",")]


def timeit(fn, reps):
    """us per launch: `reps` launches captured in one CUDA graph (no host
    launch overhead inside the events), replayed 5 times after a warm-up."""
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            for _ in range(reps):
                fn()
    torch.cuda.current_stream().wait_stream(s)
    g.replay()
    torch.cuda.synchronize()
    st = torch.cuda.current_stream()
    ts = []
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        g.replay()
        e1.record(st)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3 / reps)
    return float(np.median(ts))


def case(shape, m, reps, rows):
    dom = A.Box((0, 0, 0), tuple(s - 1 for s in shape))
    ba = A.BoxArray([dom]).max_size(m)
    dm = A.DistributionMapping.single_rank(len(ba))
    tr = A.Transport(1)
    a = A.MultiFab(ba, dm, 1, 2)
    b = A.MultiFab(ba, dm, 1, 2)
    rhs = A.MultiFab(ba, dm, 1, 1)
    gen = torch.Generator(device="cuda").manual_seed(1)
    a.storage.copy_(torch.randn(a.storage.shape, generator=gen, device="cuda", dtype=torch.float64))
    rhs.storage.copy_(torch.randn(rhs.storage.shape, generator=gen, device="cuda", dtype=torch.float64))
    A.fill_boundary(a, tr, dom, True)
    A.fill_boundary(rhs, tr, dom, True)
    dh = (65536.0,) * 3
    n = dom.num_cells()
    f = sum(2 * (e[0] * e[1] + e[1] * e[2] + e[2] * e[0]) for e in (bx.extents() for bx in ba))
    alg = 24 * n + 8 * f
    nrm = torch.zeros(1, dtype=torch.int64, device="cuda")
    cba = A.coarsened_layout(ba, 2)
    c = A.MultiFab(cba, dm, 1, 1)
    A.fill_boundary(c, tr, dom.coarsen(2), True)
    from paper_2009_12009_b200.ghosts import push_table

    tab = push_table(b, dom, True, 2)
    ops = [("sweep", 1, 0, lambda: S.gsrb_sweep(a, b, rhs, dh))]
    for cfg in CONFIGS:
        ops += [("sweep", 0, cfg, lambda: S.gsrb_sweep(a, b, rhs, dh)),
                ("sweep_prolong", 0, cfg, lambda: S.gsrb_sweep_prolong(a, b, rhs, dh, c)),
                ("sweep_norm", 0, cfg, lambda: S.gsrb_sweep_norm(a, b, rhs, dh, nrm)),
                ("sweep+push", 0, cfg, lambda: S.gsrb_sweep(a, b, rhs, dh, push=tab)),
                ("sweep_norm+push", 0, cfg, lambda: S.gsrb_sweep_norm(a, b, rhs, dh, nrm, push=tab)),
                ("sweep_prolong+push", 0, cfg, lambda: S.gsrb_sweep_prolong(a, b, rhs, dh, c, push=tab))]
    want = os.environ.get("MB_OPS")
    segs_list = [int(x) for x in os.environ.get("MB_SEGS", "0").split(",")]
    for name, kern, cfg, fn in ops:
        if want and name not in want.split(","):
            continue
        for segs in segs_list:
            try:
                with option("sweep_kernel", kern), option("stream_config", cfg), option("stream_segments", segs):
                    us = timeit(fn, reps)
            except (NotImplementedError, ValueError) as e:
                rows.append({"shape": shape, "box": m, "op": name, "kernel": kern, "error": str(e)})
                continue
            row = {"shape": list(shape), "box": m, "op": name, "kernel": ["stream", "legacy"][kern], "cfg": cfg,
                   "segs": segs, "us": round(us, 2), "alg_GBs": round(alg / us / 1e3, 1),
                   "frac": round(alg / us / 1e3 / PEAK, 3)}
            rows.append(row)
            print(json.dumps(row), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=20)
    args = ap.parse_args()
    torch.cuda.set_device(0)
    rows = []
    cases = os.environ.get("MB_CASES", "256/256,128/128,256/64,512/512,512/32")
    for c in cases.split(","):
        n, m = (int(x) for x in c.split("/"))
        shape = (n, n, n)
        case(shape, m, args.reps, rows)


if __name__ == "__main__":
    main()
