"""Host side of the device flux register (CPU): the index lists amr.FluxRegister
builds for crse_add / fine_add / reflux, applied with numpy using exactly the
kernels' formulas (csrc/amr.cu), reproduce the reference's FluxRegister bit for
bit on the hierarchies of the advection fixtures."""

import os

import numpy as np
import pytest
import torch

import paper_2009_12009_b200 as A
from paper_2009_12009_b200 import amr

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _layouts(mod, g, dim):
    bas = []
    for lev in (0, 1):
        boxes = [mod.Box(mod.IntVect(r[:dim]), mod.IntVect(r[dim:])) for r in g[f"ba{lev}"].tolist()]
        bas.append(mod.BoxArray(boxes))
    return bas


@pytest.mark.parametrize("name", ["adv2d", "adv3d"])
def test_flux_register_index_lists_match_reference(amrkit, name):
    from amrkit.coarse_fine import FluxRegister as RefFR
    from amrkit.fabarray import FabArray as RefFA

    g = np.load(os.path.join(GOLD, f"{name}.npz"))
    dim, n, nranks = (int(x) for x in g["meta"])
    ratio = tuple(int(x) for x in g["ratio"])
    rng = np.random.default_rng(11)
    rba0, rba1 = _layouts(amrkit, g, dim)
    ba0, ba1 = _layouts(A, g, dim)
    rdom = amrkit.Box(amrkit.IntVect.zero(dim), amrkit.IntVect([n - 1] * dim))
    dom = A.Box(A.IntVect([0] * dim), A.IntVect([n - 1] * dim))

    def fluxes(ba):
        return {i: [rng.standard_normal((1,) + tuple(e + (1 if k == d else 0) for k, e in enumerate(ba[i].extents())))
                    for d in range(dim)] for i in range(len(ba))}

    cfl, ffl = fluxes(rba0), fluxes(rba1)
    dtdx = [0.37 + 0.1 * d for d in range(dim)]

    # reference
    ref = RefFR(rba1, amrkit.IntVect(ratio), ncomp=1).zero()
    ref.crse_add(cfl, rba0, rdom, scale=1.0)
    for k in range(len(rba1)):
        ref.fine_add(k, ffl[k], scale=0.5)
    rcrse = RefFA(rba0, amrkit.DistributionMapping.single_rank(len(rba0)), 1, 1)
    init = {i: rng.standard_normal(rcrse.fab(i).valid().shape) for i in range(len(rba0))}
    for i in range(len(rba0)):
        rcrse.fab(i).valid()[...] = init[i]
    ref.reflux(rcrse, dtdx, rdom, (True,) * dim)

    # device register's index lists, applied with the kernels' formulas
    dm0 = A.DistributionMapping.single_rank(len(ba0))
    dm1 = A.DistributionMapping.single_rank(len(ba1))
    cfa = A.FabArray(ba0, dm0, 1, 1, device="cpu")
    ffa = A.FabArray(ba1, dm1, 1, 1, device="cpu")
    cf, ff = amr.FaceFluxes(cfa), amr.FaceFluxes(ffa)
    for i in range(len(ba0)):
        for d in range(dim):
            cf.box(i, d).copy_(torch.as_tensor(cfl[i][d]))
    for i in range(len(ba1)):
        for d in range(dim):
            ff.box(i, d).copy_(torch.as_tensor(ffl[i][d]))
    fr = amr.FluxRegister(ba1, ratio, 1, device="cpu")
    reg = np.zeros(fr.size)
    for d in range(dim):
        pr = fr._crse_pairs(cf, ba0, dom, d).numpy().reshape(-1, 2)
        F = cf.data[d].numpy()
        for p0, p1 in pr:  # reg[p0] = reg[p0] - scale * F[p1]
            reg[p0] = reg[p0] - 1.0 * F[p1]
    for d, nsrc, seq, idx in fr._fine_lists(ff, None):
        F = ff.data[d].numpy()
        for e in idx.numpy().reshape(-1, 1 + nsrc):
            a = [F[x] for x in e[1:]]
            if nsrc == 2:
                avg = (a[0] + a[1]) / 2.0
            elif nsrc == 4:
                avg = ((((a[0] + a[1]) + a[2]) + a[3]) if seq else ((a[0] + a[1]) + (a[2] + a[3]))) / 4.0
            else:
                avg = a[0]
            reg[e[0]] = reg[e[0]] + 0.5 * avg
    for k in range(len(ba1)):
        for d in range(dim):
            for side in ("lo", "hi"):
                want = ref.patches[(k, d, side)]["data"]
                p = [i for i, (kk, dd, ss, _, _) in enumerate(fr.patches) if (kk, dd, ss) == (k, d, side)][0]
                got = reg[fr.poff[p] : fr.poff[p] + want.size].reshape(want.shape)
                assert np.array_equal(got, want), (k, d, side)
    # reflux onto the same coarse data
    for i in range(len(ba0)):
        cfa.fab(i).valid().copy_(torch.as_tensor(init[i]))
    tgt, start, src, sign, dims = fr._reflux_plan(cfa, dom, (True,) * dim)
    crse = cfa.storage.numpy()
    tgt, start, src = tgt.numpy(), start.numpy(), src.numpy()
    coef = [sign[e] * float(dtdx[dims[e]]) for e in range(len(sign))]
    for t in range(len(tgt)):
        v = crse[tgt[t]]
        for e in range(start[t], start[t + 1]):
            v = v + coef[e] * reg[src[e]]
        crse[tgt[t]] = v
    for i in range(len(ba0)):
        assert np.array_equal(cfa.fab(i).valid().numpy(), rcrse.fab(i).valid()), i
