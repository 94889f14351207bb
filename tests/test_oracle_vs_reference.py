"""Pin the oracle restatement against the reference itself (amrkit from
/root/reference, build container only; skipped elsewhere) and against the
committed golden fixtures generated from it (everywhere)."""

import glob
import os

import numpy as np
import pytest

from oracle import mesh_ref as M

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _ref_cover(ak, rng, dom, nsplits):
    boxes = [dom]
    for _ in range(nsplits):
        i = int(rng.integers(len(boxes)))
        b = boxes[i]
        e = b.extents()
        axes = [d for d in range(b.dim) if e[d] >= 2]
        if not axes:
            continue
        d = axes[int(rng.integers(len(axes)))]
        cut = b.lo[d] + int(rng.integers(1, e[d]))
        hi = list(b.hi.coords)
        hi[d] = cut - 1
        lo = list(b.lo.coords)
        lo[d] = cut
        boxes[i : i + 1] = [ak.Box(b.lo, ak.IntVect(hi)), ak.Box(ak.IntVect(lo), b.hi)]
    return ak.BoxArray(boxes)


def _t(b):
    return (b.lo.coords, b.hi.coords)


def test_oracle_fill_copy_sum_reduce_match_amrkit(amrkit, rng):
    from amrkit.distribution import default_costs, sfc_distribute
    from amrkit.fabarray import FabArray, build_plan_fill_boundary, fill_boundary, parallel_copy, reduce, sum_boundary

    ak = amrkit
    for trial in range(10):
        dim = 2 + trial % 2
        n = int(rng.integers(8, 16))
        dom = ak.Box(ak.IntVect([0] * dim), ak.IntVect([n - 1] * dim))
        ba = _ref_cover(ak, rng, dom, int(rng.integers(3, 8)))
        nr = int(rng.integers(1, 4))
        per = tuple(bool(rng.integers(0, 2)) for _ in range(dim))
        ng, nc = int(rng.integers(1, 3)), int(rng.integers(1, 3))
        fa = FabArray(ba, sfc_distribute(ba, default_costs(ba), nr), nc, ng)
        for i in range(len(ba)):
            fa.fab(i).data[...] = rng.normal(size=fa.fab(i).data.shape)
        boxes = [_t(b) for b in ba]
        d = _t(dom)
        # plan records
        plan = build_plan_fill_boundary(ba, ng, dom, per)
        want = [(r.src_index, r.dst_index, _t(r.src_box), r.shift.coords) for r in plan.records]
        assert want == M.fill_records(boxes, ng, d, per)
        # fill
        of = {i: fa.fab(i).data.copy() for i in range(len(ba))}
        fill_boundary(fa, ak.Transport(nr), dom, per)
        M.fill_boundary(boxes, of, ng, d, per)
        for i in range(len(ba)):
            assert np.array_equal(of[i], fa.fab(i).data)
        # sum
        of = {i: fa.fab(i).data.copy() for i in range(len(ba))}
        sum_boundary(fa, ak.Transport(nr), dom, per)
        M.sum_boundary(boxes, of, ng, d, per)
        for i in range(len(ba)):
            assert np.array_equal(of[i], fa.fab(i).data)
        # reduce (per-box numpy, rank-ordered fold: bit-identical)
        for kind in ("sum", "min", "max"):
            got = reduce(fa, kind, nc - 1, ak.Transport(nr))
            owner = list(fa.dm.owner)
            assert got == M.reduce(boxes, of, ng, kind, nc - 1, owner, nr)
        # parallel_copy onto another cover, periodic images included
        dba = _ref_cover(ak, rng, dom, 4)
        dfa = FabArray(dba, sfc_distribute(dba, default_costs(dba), nr), nc, 1)
        parallel_copy(dfa, fa, ak.Transport(nr), dom, per)
        od = {i: np.zeros_like(dfa.fab(i).data) for i in range(len(dba))}
        M.parallel_copy([_t(b) for b in dba], od, 1, boxes, of, ng, d, per)
        for i in range(len(dba)):
            assert np.array_equal(od[i][(slice(None),) + M.region_index(_t(dba[i]), 1, _t(dba[i]))], dfa.fab(i).valid())


def test_oracle_interlevel_match_amrkit(amrkit, rng):
    from amrkit.coarse_fine import average_down, interp_to_fine
    from amrkit.distribution import DistributionMapping
    from amrkit.fabarray import FabArray

    ak = amrkit
    for dim in (2, 3):
        fba = ak.BoxArray([ak.Box(ak.IntVect([4] * dim), ak.IntVect([11] * dim)),
                           ak.Box(ak.IntVect([12] + [4] * (dim - 1)), ak.IntVect([19] + [11] * (dim - 1)))])
        cba = ak.BoxArray([ak.Box(ak.IntVect([0] * dim), ak.IntVect([11] + [7] * (dim - 1)))])
        fine = FabArray(fba, DistributionMapping.single_rank(2), 2, 0)
        crse = FabArray(cba, DistributionMapping.single_rank(1), 2, 1)
        ff = {i: rng.normal(size=fine.fab(i).data.shape) for i in range(2)}
        for i in range(2):
            fine.fab(i).data[...] = ff[i]
        crse.fab(0).data[...] = -3.0
        cf = {0: crse.fab(0).data.copy()}
        average_down(fine, crse, ak.IntVect([2] * dim), ak.Transport(1))
        r = (2,) * dim
        M.average_down([_t(b) for b in fba], ff, 0, [_t(b) for b in cba], cf, 1, r)
        assert np.array_equal(cf[0], crse.fab(0).data)
        crse.fab(0).data[...] = rng.normal(size=crse.fab(0).data.shape)
        cf = {0: crse.fab(0).data.copy()}
        interp_to_fine(fine, crse, ak.IntVect([2] * dim), ak.Transport(1), method="pc")
        of = {i: np.zeros((2,) + tuple(M.ext(_t(fba[i])))) for i in range(2)}
        M.interp_pc([_t(b) for b in fba], of, 0, [_t(b) for b in cba], cf, 1, r)
        for i in range(2):
            assert np.array_equal(of[i], fine.fab(i).data)


def test_oracle_matches_golden_fixtures():
    files = sorted(glob.glob(os.path.join(GOLDEN, "mesh_case*.npz")))
    assert files
    for f in files:
        z = np.load(f)
        dim = int(z["dim"])
        boxes = [(tuple(r[:dim].tolist()), tuple(r[dim:].tolist())) for r in z["boxes"]]
        dom = (tuple(z["domain"][:dim].tolist()), tuple(z["domain"][dim:].tolist()))
        per = tuple(bool(p) for p in z["periodic"])
        ng, nc = int(z["ngrow"]), int(z["ncomp"])
        assert np.array_equal(M.records_table(M.fill_records(boxes, ng, dom, per)), z["plan"])
        fabs = M.make_fabs(boxes, nc, ng, -7777.0)
        M.load_global(boxes, fabs, ng, dom, z["g"])
        M.fill_boundary(boxes, fabs, ng, dom, per)
        assert np.array_equal(np.concatenate([fabs[i].ravel() for i in range(len(boxes))]), z["filled"])
        owner = z["owner"].tolist()
        red = [M.reduce(boxes, fabs, ng, k, nc - 1, owner, int(z["nranks"])) for k in ("sum", "min", "max")]
        assert red == list(z["reduce"])
        sin = z["sum_in"]
        off = 0
        for i in range(len(boxes)):
            nn = fabs[i].size
            fabs[i] = sin[off : off + nn].reshape(fabs[i].shape).copy()
            off += nn
        M.sum_boundary(boxes, fabs, ng, dom, per)
        assert np.array_equal(np.concatenate([fabs[i].ravel() for i in range(len(boxes))]), z["sum_out"])


def test_oracle_matches_golden_domain_bc():
    z = np.load(os.path.join(GOLDEN, "domain_bc.npz"))
    boxes = [(tuple(r[:2].tolist()), tuple(r[2:].tolist())) for r in z["boxes"]]
    fabs = {0: z["in0"].copy(), 1: z["in1"].copy()}
    M.apply_domain_boundary(boxes, fabs, 2, ((0, 0), (7, 9)), ("external", "extrap"), ("extrap", "external"), -1.5)
    assert np.array_equal(fabs[0], z["out0"]) and np.array_equal(fabs[1], z["out1"])
