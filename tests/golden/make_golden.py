"""Generate golden fixtures for the mesh path from the REFERENCE itself.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

It imports the unmodified reference package ``amrkit`` from
/root/reference/pkg/src, runs fill_boundary / parallel_copy / sum_boundary /
reduce / average_down / interp_to_fine('pc') / apply_domain_boundary on seeded
layouts, and stores inputs + outputs (plus the fill-plan record tables) in
small .npz files next to this script.  The GPU box has no /root/reference;
tests there compare the device path against these fixtures and the oracle.
"""

from __future__ import annotations

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))


def _boxes(ba):
    return np.array([tuple(b.lo) + tuple(b.hi) for b in ba], dtype=np.int32)


def _random_cover(rng, Box, IntVect, BoxArray, domain, nsplits):
    boxes = [domain]
    for _ in range(nsplits):
        i = int(rng.integers(len(boxes)))
        b = boxes[i]
        e = b.extents()
        axes = [d for d in range(b.dim) if e[d] >= 2]
        if not axes:
            continue
        d = axes[int(rng.integers(len(axes)))]
        cut = b.lo[d] + int(rng.integers(1, e[d]))
        a_hi = list(b.hi.coords)
        a_hi[d] = cut - 1
        b_lo = list(b.lo.coords)
        b_lo[d] = cut
        boxes[i : i + 1] = [Box(b.lo, IntVect(a_hi)), Box(IntVect(b_lo), b.hi)]
    return BoxArray(boxes)


def main():
    sys.path.insert(0, REF)
    import amrkit
    from amrkit import Box, BoxArray, IntVect, Transport
    from amrkit.amr_core import BoundaryRecord, Geometry, apply_domain_boundary
    from amrkit.coarse_fine import average_down, interp_to_fine
    from amrkit.distribution import default_costs, sfc_distribute
    from amrkit.fabarray import (
        FabArray,
        build_plan_fill_boundary,
        fill_boundary,
        parallel_copy,
        reduce,
        sum_boundary,
    )

    def rec_table(plan, dim):
        t = np.zeros((len(plan.records), 11), dtype=np.int32)
        pad = 3 - dim
        for r, rec in enumerate(plan.records):
            t[r, 0] = rec.src_index
            t[r, 1] = rec.dst_index
            t[r, 2 + pad : 5] = rec.src_box.lo.coords
            t[r, 5 + pad : 8] = rec.src_box.hi.coords
            t[r, 8 + pad : 11] = rec.shift.coords
        return t

    def fabs_flat(fa):
        return np.concatenate([fa.fab(i).data.ravel() for i in range(len(fa.ba))])

    rng = np.random.default_rng(20261018)
    cases = []
    # fill / copy / sum on random covers, 2-D and 3-D, mixed periodicity
    for case in range(8):
        dim = 2 if case % 2 == 0 else 3
        n = int(rng.integers(10, 18))
        domain = Box(IntVect.zero(dim), IntVect([n - 1] * dim))
        ba = _random_cover(rng, Box, IntVect, BoxArray, domain, int(rng.integers(4, 8)))
        nranks = int(rng.integers(1, 5))
        periodic = tuple(bool(rng.integers(0, 2)) for _ in range(dim))
        ngrow = int(rng.integers(1, 3))
        ncomp = int(rng.integers(1, 3))
        dm = sfc_distribute(ba, default_costs(ba), nranks)
        fa = FabArray(ba, dm, ncomp, ngrow)
        g = rng.normal(size=(ncomp,) + tuple(domain.extents()))
        for i in range(len(ba)):
            f = fa.fab(i)
            f.data[...] = -7777.0
            b = ba[i]
            sel = tuple(slice(b.lo[d], b.hi[d] + 1) for d in range(dim))
            f.valid()[...] = g[(slice(None),) + sel]
        fill_boundary(fa, Transport(nranks), domain, periodic)
        plan = build_plan_fill_boundary(ba, ngrow, domain, periodic)
        filled = fabs_flat(fa)
        # sum_boundary on every stored cell randomised
        sfa = FabArray(ba, dm, ncomp, ngrow)
        sin = []
        for i in range(len(ba)):
            v = rng.normal(size=sfa.fab(i).data.shape)
            sfa.fab(i).data[...] = v
            sin.append(v.ravel())
        sum_boundary(sfa, Transport(nranks), domain, periodic)
        # parallel_copy onto another random cover (with periodic images)
        dba = _random_cover(rng, Box, IntVect, BoxArray, domain, int(rng.integers(3, 7)))
        dfa = FabArray(dba, sfc_distribute(dba, default_costs(dba), nranks), ncomp, 1)
        for i in range(len(dba)):
            dfa.fab(i).data[...] = 0.0
        parallel_copy(dfa, fa, Transport(nranks), domain, periodic)
        red = [reduce(fa, k, ncomp - 1, Transport(nranks)) for k in ("sum", "min", "max")]
        cases.append(
            dict(
                dim=dim,
                domain=np.array(tuple(domain.lo) + tuple(domain.hi), dtype=np.int32),
                boxes=_boxes(ba),
                owner=np.array(dm.owner, dtype=np.int32),
                nranks=nranks,
                periodic=np.array(periodic, dtype=np.uint8),
                ngrow=ngrow,
                ncomp=ncomp,
                g=g,
                filled=filled,
                plan=rec_table(plan, dim),
                sum_in=np.concatenate(sin),
                sum_out=fabs_flat(sfa),
                dst_boxes=_boxes(dba),
                copy_out=fabs_flat(dfa),
                reduce=np.array(red),
            )
        )
    for k, c in enumerate(cases):
        np.savez_compressed(os.path.join(HERE, f"mesh_case{k}.npz"), **c)

    # inter-level: average_down / interp pc on a 3-D two-box fine layout
    fine_ba = BoxArray([Box(IntVect(4, 4, 4), IntVect(11, 11, 11)), Box(IntVect(12, 4, 4), IntVect(19, 11, 11))])
    crse_ba = BoxArray([Box(IntVect(0, 0, 0), IntVect(11, 7, 7))])
    one = lambda ba: sfc_distribute(ba, default_costs(ba), 1)  # noqa: E731
    fine = FabArray(fine_ba, one(fine_ba), 1, 0)
    crse = FabArray(crse_ba, one(crse_ba), 1, 1)
    fv = [rng.normal(size=fine.fab(i).data.shape) for i in range(2)]
    for i in range(2):
        fine.fab(i).data[...] = fv[i]
    crse.fab(0).data[...] = -3.0
    average_down(fine, crse, IntVect(2, 2, 2), Transport(1))
    avg_out = crse.fab(0).data.copy()
    cv = rng.normal(size=crse.fab(0).data.shape)
    crse.fab(0).data[...] = cv
    interp_to_fine(fine, crse, IntVect(2, 2, 2), Transport(1), method="pc")
    np.savez_compressed(
        os.path.join(HERE, "interlevel.npz"),
        fine_boxes=_boxes(fine_ba),
        crse_boxes=_boxes(crse_ba),
        fine_in0=fv[0],
        fine_in1=fv[1],
        avg_out=avg_out,
        crse_in=cv,
        interp_out0=fine.fab(0).data.copy(),
        interp_out1=fine.fab(1).data.copy(),
    )

    # domain boundary fill (2-D, external + extrap), cf. tests/test_amr_core.py:180-192
    geom = Geometry(Box(IntVect(0, 0), IntVect(7, 9)), (0.0, 0.0), (1.0, 1.0), False)
    ba = BoxArray([Box(IntVect(0, 0), IntVect(3, 9)), Box(IntVect(4, 0), IntVect(7, 9))])
    fa = FabArray(ba, sfc_distribute(ba, default_costs(ba), 1), 1, 2)
    ins = []
    for i in range(2):
        v = rng.normal(size=fa.fab(i).data.shape)
        fa.fab(i).data[...] = v
        ins.append(v)
    rec = BoundaryRecord(("external", "extrap"), ("extrap", "external"), external_value=-1.5)
    apply_domain_boundary(fa, geom, rec)
    np.savez_compressed(
        os.path.join(HERE, "domain_bc.npz"),
        boxes=_boxes(ba),
        in0=ins[0],
        in1=ins[1],
        out0=fa.fab(0).data.copy(),
        out1=fa.fab(1).data.copy(),
    )
    _plotfile_golden()
    _advection_golden()
    print("amrkit", amrkit.__version__, "->", HERE)


ADV_CASES = [
    # name, dim, n, max_grid, blocking, velocity, nranks, cfl, steps
    ("adv2d", 2, 16, 8, 4, (1.0, 0.5), 2, 0.4, (1, 5, 100)),
    ("adv3d", 3, 16, 8, 4, (1.0, 0.5, 0.25), 2, 0.4, (1, 4)),
]


def _advection_golden():
    """Two-level subcycled advection (advect.py:130-188) run by the reference:
    the hierarchy its regrid built, the initial state and the state after a few
    coarse steps, with and without refluxing."""
    from amrkit.advect import AdvectionSolver
    from amrkit.amr_core import Geometry, GridGenParams

    import amrkit

    for name, dim, n, mg, bf, vel, nranks, cfl, steps in ADV_CASES:
        out = {}
        for reflux in (True, False):
            domain = amrkit.Box(amrkit.IntVect.zero(dim), amrkit.IntVect([n - 1] * dim))
            geom = Geometry(domain, (0.0,) * dim, (1.0,) * dim, (True,) * dim)
            params = GridGenParams(dim=dim, max_level=1, max_grid_size=mg, blocking_factor=bf)
            s = AdvectionSolver(geom, params, velocity=vel, nranks=nranks, cfl=cfl, use_reflux=reflux,
                                regrid_interval=0)
            assert s.hier.finest_level == 1
            tag = "r" if reflux else "n"
            if reflux:
                for lev in (0, 1):
                    out[f"ba{lev}"] = _boxes(s.hier.ba(lev))
                    out[f"dm{lev}"] = np.array(list(s.hier.dm(lev)), dtype=np.int32)
                out["ratio"] = np.array(s.params.ref_ratio[0].coords, dtype=np.int32)
                out["mass0"] = np.array(s.total_mass())
            done = 0
            for st in (0,) + tuple(steps):
                while done < st:
                    s.step()
                    done += 1
                for lev in (0, 1):
                    fa = s.hier.field("phi", lev)
                    for i in range(len(fa.ba)):
                        out[f"{tag}_s{st}_L{lev}_b{i}"] = fa.fab(i).valid().copy()
                out[f"{tag}_s{st}_mass"] = np.array(s.total_mass())
                out[f"{tag}_s{st}_time"] = np.array(s.time)
        out["steps"] = np.array((0,) + tuple(steps))
        out["meta"] = np.array([dim, n, nranks], dtype=np.int32)
        out["velocity"] = np.array(vel)
        out["cfl"] = np.array(cfl)
        np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **out)


def _plotfile_golden():
    """Directory digests + Header text of amrkit.write_plotfile for the cases
    in plotfile_cases.py (the device writer must reproduce them byte for byte)."""
    import json
    import tempfile
    import types

    import amrkit
    from amrkit import distribution, plotfile

    sys.path.insert(0, HERE)
    import plotfile_cases as PC

    ns = types.SimpleNamespace(
        Box=amrkit.Box, IntVect=amrkit.IntVect, BoxArray=amrkit.BoxArray, Geometry=amrkit.Geometry,
        FabArray=amrkit.FabArray, sfc_distribute=distribution.sfc_distribute,
        default_costs=distribution.default_costs, PlotfileHeader=plotfile.PlotfileHeader)
    out = {}
    for case in PC.CASES:
        header, meshes = PC.build(ns, case)
        with tempfile.TemporaryDirectory() as tmp:
            path = os.path.join(tmp, "plt")
            plotfile.write_plotfile(path, meshes, header).wait()
            with open(os.path.join(path, "Header")) as fh:
                text = fh.read()
            out[case[0]] = {"digest": PC.dir_digest(path), "header": text}
    with open(os.path.join(HERE, "plotfile.json"), "w") as fh:
        json.dump(out, fh, indent=1)


if __name__ == "__main__":
    main()
