"""Plotfile golden cases shared by make_golden.py (run against the reference)
and tests/test_gpu_plotfile.py (run against the device writer): layouts and
cell values are a pure function of the case parameters (explicit seeds)."""

import hashlib
import os

import numpy as np

# (name, dim, n, max_size, ncomp, nranks, two_levels, time, names)
CASES = [
    ("two_level_2d", 2, 16, 8, 2, 1, True, 0.625, ["density", "tracer"]),
    ("two_level_2d_r4", 2, 16, 8, 2, 4, True, 0.625, ["density", "tracer"]),
    ("boxes_3d_r3", 3, 32, 16, 1, 3, False, 1.5, ["phi"]),
]


def values(lev, g, c, extents):
    return np.random.default_rng(100003 * lev + 101 * g + c).normal(size=tuple(extents))


def build(mod, case):
    """(header, meshes) with the package `mod` (amrkit or paper_2009_12009_b200)."""
    name, dim, n, m, ncomp, nranks, two, time, names = case
    Box, IntVect, BoxArray = mod.Box, mod.IntVect, mod.BoxArray
    domain = Box(IntVect([0] * dim), IntVect([n - 1] * dim))
    geom0 = mod.Geometry(domain, (0.0,) * dim, (1.0,) * dim, (True,) * dim)
    levels = [(BoxArray([domain]).max_size(m), geom0)]
    if two:
        fine = Box(IntVect([n // 2] * dim), IntVect([n + n // 2 - 1] * dim))
        levels.append((BoxArray([fine]).max_size(m), geom0.refine(IntVect([2] * dim))))
    meshes = []
    for lev, (ba, _) in enumerate(levels):
        dm = mod.sfc_distribute(ba, mod.default_costs(ba), nranks)
        fa = mod.FabArray(ba, dm, ncomp, 0)
        for g in range(len(ba)):
            for c in range(ncomp):
                v = values(lev, g, c, ba[g].extents())
                tgt = fa.fab(g).valid(c)
                if hasattr(tgt, "copy_"):  # device Fab (torch view)
                    import torch

                    tgt.copy_(torch.as_tensor(v))
                else:
                    tgt[...] = v
        meshes.append(fa)
    header = mod.PlotfileHeader(time, names, [g for _, g in levels]) if hasattr(mod, "PlotfileHeader") else None
    return header, meshes


def dir_digest(path):
    """Same digest as the reference's tests (test_plotfile.py:36-45)."""
    h = hashlib.sha256()
    for root, dirs, files in os.walk(path):
        dirs.sort()
        for fname in sorted(files):
            full = os.path.join(root, fname)
            h.update(os.path.relpath(full, path).encode())
            with open(full, "rb") as fh:
                h.update(fh.read())
    return h.hexdigest()
