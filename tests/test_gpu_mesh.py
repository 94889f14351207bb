"""Device ghost exchange / copy / fold / reduce / inter-level ops vs the oracle
and the reference's golden outputs.  Bar: bit-exact."""

import glob
import os

import numpy as np
import pytest
import torch

import paper_2009_12009_b200 as A
from paper_2009_12009_b200 import counters
from oracle import mesh_ref as M
from helpers import load_device_from_oracle, oracle_fabs_from_device, random_cover, tboxes, wrap

pytestmark = pytest.mark.gpu
GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _make(rng, dim, nranks, ngrow=2, ncomp=2, n=None):
    n = n or int(rng.integers(12, 24))
    dom = A.Box([0] * dim, [n - 1] * dim)
    ba = random_cover(rng, dom, nsplits=int(rng.integers(4, 9)))
    dm = A.sfc_distribute(ba, A.default_costs(ba), nranks)
    return dom, A.MultiFab(ba, dm, ncomp, ngrow)


def _sentinel_load(fa, dom, g, sentinel=-7777.0):
    fa.setval(sentinel)
    fa.load_valid_from(dom, g)


def test_fill_boundary_matches_dense_wrap_oracle(rng):
    for dim in (2, 3):
        for _ in range(4):
            nranks = int(rng.integers(1, 5))
            per = tuple(bool(rng.integers(0, 2)) for _ in range(dim))
            dom, fa = _make(rng, dim, nranks)
            g = rng.normal(size=(fa.ncomp,) + tuple(dom.extents()))
            _sentinel_load(fa, dom, g)
            A.fill_boundary(fa, A.Transport(nranks), dom, per)
            torch.cuda.synchronize()
            for i, fab in fa.fabs.items():
                data = fab.data.cpu().numpy()
                for cell in fab.gbox.cells():
                    if fa.ba[i].contains(cell):
                        continue
                    src = wrap(cell, dom, per)
                    loc = tuple(cell[d] - fab.gbox.lo[d] for d in range(dim))
                    got = data[(slice(None),) + loc]
                    if src is None:
                        assert np.all(got == -7777.0)
                    else:
                        assert np.array_equal(got, g[(slice(None),) + src])


@pytest.mark.parametrize("shape,ngrow,width,ncomp", [((16, 16, 16), 2, 2, 1), ((16, 12, 20), 2, 1, 2),
                                                     ((8, 10, 6), 3, 3, 1), ((32, 8, 64), 2, 2, 2),
                                                     ((6, 6, 6), 1, 1, 3)])
def test_single_periodic_box_fill_matches_plan_and_oracle(rng, shape, ngrow, width, ncomp):
    """One box = the whole periodic domain takes the record-free wrap kernel
    (amrb_fill_wrap); it leaves every cell -- ghosts beyond the fill width
    included -- exactly as the fill-plan copy program and as the dense-wrap
    oracle."""
    from paper_2009_12009_b200 import comm
    from paper_2009_12009_b200.plans import build_plan_fill_boundary

    dom = A.Box((0, 0, 0), tuple(e - 1 for e in shape))
    ba = A.BoxArray([dom])
    dm = A.DistributionMapping.single_rank(1)
    g = rng.normal(size=(ncomp,) + shape)
    tr = A.Transport(1)
    a = A.MultiFab(ba, dm, ncomp, ngrow)
    b = A.MultiFab(ba, dm, ncomp, ngrow)
    for f in (a, b):
        _sentinel_load(f, dom, g)
    assert comm._single_periodic_box(a, tr, dom, True, False)
    A.fill_boundary(a, tr, dom, True, ngrow=width)
    comm._execute(build_plan_fill_boundary(ba, width, dom, True), b, b, tr, 0)  # the copy program
    torch.cuda.synchronize()
    assert torch.equal(a.fab(0).data, b.fab(0).data)
    data = a.fab(0).data.cpu().numpy()
    fab = a.fab(0)
    for cell in fab.gbox.cells():
        loc = tuple(cell[d] - fab.gbox.lo[d] for d in range(3))
        if all(-width <= cell[d] < shape[d] + width for d in range(3)):
            src = tuple(cell[d] % shape[d] for d in range(3))
            assert np.array_equal(data[(slice(None),) + loc], g[(slice(None),) + src])
        else:
            assert np.all(data[(slice(None),) + loc] == -7777.0)


def test_fill_boundary_equals_oracle_executor(rng):
    for dim in (1, 2, 3):
        for _ in range(3):
            dom, fa = _make(rng, dim, 1, ngrow=int(rng.integers(1, 4)), ncomp=int(rng.integers(1, 3)))
            per = tuple(bool(rng.integers(0, 2)) for _ in range(dim))
            fabs = M.make_fabs(tboxes(fa.ba), fa.ncomp, fa.ngrow)
            for f in fabs.values():
                f[...] = rng.normal(size=f.shape)
            load_device_from_oracle(fa, fabs)
            M.fill_boundary(tboxes(fa.ba), fabs, fa.ngrow, (tuple(dom.lo), tuple(dom.hi)), per)
            A.fill_boundary(fa, A.Transport(1), dom, per)
            got = oracle_fabs_from_device(fa)
            for i in fabs:
                assert np.array_equal(got[i], fabs[i])


def test_fill_boundary_partial_width(rng):
    dom, fa = _make(rng, 3, 1, ngrow=2, ncomp=1)
    fabs = M.make_fabs(tboxes(fa.ba), 1, 2)
    for f in fabs.values():
        f[...] = rng.normal(size=f.shape)
    load_device_from_oracle(fa, fabs)
    M.fill_boundary(tboxes(fa.ba), fabs, 2, (tuple(dom.lo), tuple(dom.hi)), (True,) * 3, width=1)
    A.fill_boundary(fa, A.Transport(1), dom, True, ngrow=1)
    got = oracle_fabs_from_device(fa)
    for i in fabs:
        assert np.array_equal(got[i], fabs[i])


def test_fill_boundary_bit_identical_across_ranks(rng):
    dom, base = _make(rng, 2, 1, n=20)
    g = rng.normal(size=(base.ncomp,) + tuple(dom.extents()))
    results = []
    for nranks in (1, 2, 4, 8):
        dm = A.sfc_distribute(base.ba, A.default_costs(base.ba), nranks)
        fa = A.MultiFab(base.ba, dm, base.ncomp, base.ngrow)
        fa.load_valid_from(dom, g)
        A.fill_boundary(fa, A.Transport(nranks), dom, (True, True))
        results.append(oracle_fabs_from_device(fa))
    for other in results[1:]:
        for i in other:
            assert np.array_equal(results[0][i], other[i])


def test_one_message_per_rank_pair(rng):
    nranks = 4
    dom, fa = _make(rng, 2, nranks, n=24)
    fa.load_valid_from(dom, rng.normal(size=(fa.ncomp,) + tuple(dom.extents())))
    plan = A.build_plan_fill_boundary(fa.ba, fa.ngrow, dom, (True, True))
    pairs = {(s, d) for (s, d) in plan.pairs(fa.dm, fa.dm) if s != d}
    counters.reset("transport_messages", "transport_bytes")
    A.fill_boundary(fa, A.Transport(nranks), dom, (True, True))
    assert counters.get("transport_messages") == len(pairs)
    t = plan.table()
    remote = [r for r in range(len(t)) if fa.dm[t[r, 0]] != fa.dm[t[r, 1]]]
    cells = sum(int(np.prod(t[r, 5:8] - t[r, 2:5] + 1)) for r in remote)
    assert counters.get("transport_bytes") == 8 * fa.ncomp * cells


def test_parallel_copy_matches_oracle(rng):
    for dim in (2, 3):
        nranks = int(rng.integers(1, 5))
        dom = A.Box([0] * dim, [15] * dim)
        sba, dba = random_cover(rng, dom, 5), random_cover(rng, dom, 7)
        src = A.MultiFab(sba, A.sfc_distribute(sba, A.default_costs(sba), nranks), 2, 1)
        dst = A.MultiFab(dba, A.sfc_distribute(dba, A.default_costs(dba), nranks), 2, 1)
        g = rng.normal(size=(2,) + tuple(dom.extents()))
        src.load_valid_from(dom, g)
        dst.setval(0.0)
        A.parallel_copy(dst, src, A.Transport(nranks), dom)
        for i, f in dst.fabs.items():
            b = dba[i]
            want = g[(slice(None),) + tuple(slice(b.lo[d], b.hi[d] + 1) for d in range(dim))]
            assert np.array_equal(f.valid().cpu().numpy(), want)


def test_sum_boundary_matches_oracle_bitwise(rng):
    for dim in (2, 3):
        nranks = int(rng.integers(1, 4))
        dom, fa = _make(rng, dim, nranks, ngrow=1, ncomp=1, n=12)
        per = (True,) * dim
        fabs = M.make_fabs(tboxes(fa.ba), 1, 1)
        for f in fabs.values():
            f[...] = rng.normal(size=f.shape)
        load_device_from_oracle(fa, fabs)
        M.sum_boundary(tboxes(fa.ba), fabs, 1, (tuple(dom.lo), tuple(dom.hi)), per)
        A.sum_boundary(fa, A.Transport(nranks), dom, per)
        got = oracle_fabs_from_device(fa)
        for i in fabs:
            assert np.array_equal(got[i], fabs[i])


def test_reduce_matches_numpy(rng):
    dom, fa = _make(rng, 2, 4, ncomp=2)
    g = rng.normal(size=(2,) + tuple(dom.extents()))
    fa.load_valid_from(dom, g)
    tr = A.Transport(4)
    assert np.isclose(A.reduce(fa, "sum", 0, tr), g[0].sum(), rtol=1e-13)
    assert A.reduce(fa, "min", 1, tr) == g[1].min()
    assert A.reduce(fa, "max", 1, tr) == g[1].max()
    with pytest.raises(ValueError):
        A.reduce(fa, "median", 0, tr)


def test_gather_global_round_trip(rng):
    dom, fa = _make(rng, 3, 2, ncomp=1)
    g = rng.normal(size=(1,) + tuple(dom.extents()))
    fa.load_valid_from(dom, g)
    assert np.array_equal(A.gather_global(fa, dom, 0), g[0])


def test_plan_and_program_reuse(rng):
    dom, fa = _make(rng, 2, 2)
    tr = A.Transport(2)
    A.plan_cache_clear()
    counters.reset("plans_built")
    A.fill_boundary(fa, tr, dom, (True, True))
    built = counters.get("plans_built")
    A.fill_boundary(fa, tr, dom, (True, True))
    assert counters.get("plans_built") == built
    assert len(fa._progs) == 1


def _golden_layout(z):
    dim = int(z["dim"])
    boxes = [A.Box(r[:dim].tolist(), r[dim:].tolist()) for r in z["boxes"]]
    dom = A.Box(z["domain"][:dim].tolist(), z["domain"][dim:].tolist())
    ba = A.BoxArray(boxes)
    dm = A.DistributionMapping(z["owner"].tolist(), int(z["nranks"]))
    return dim, dom, ba, dm


def _flat(fa):
    return np.concatenate([fa.fab(i).data.cpu().numpy().ravel() for i in range(len(fa.ba))])


def _load_flat(fa, flat):
    off = 0
    for i in range(len(fa.ba)):
        f = fa.fab(i)
        n = f.data.numel()
        f.data.copy_(torch.as_tensor(flat[off : off + n].reshape(tuple(f.data.shape))))
        off += n


def test_reference_golden_fill_sum_copy_reduce():
    files = sorted(glob.glob(os.path.join(GOLDEN, "mesh_case*.npz")))
    assert files
    for f in files:
        z = np.load(f)
        dim, dom, ba, dm = _golden_layout(z)
        nr = int(z["nranks"])
        per = tuple(bool(p) for p in z["periodic"])
        ng, nc = int(z["ngrow"]), int(z["ncomp"])
        fa = A.MultiFab(ba, dm, nc, ng)
        fa.setval(-7777.0)
        fa.load_valid_from(dom, z["g"])
        A.fill_boundary(fa, A.Transport(nr), dom, per)
        assert np.array_equal(_flat(fa), z["filled"]), f
        red = [A.reduce(fa, k, nc - 1, A.Transport(nr)) for k in ("sum", "min", "max")]
        assert np.isclose(red[0], z["reduce"][0], rtol=1e-13) and red[1:] == list(z["reduce"][1:])
        sfa = A.MultiFab(ba, dm, nc, ng)
        _load_flat(sfa, z["sum_in"])
        A.sum_boundary(sfa, A.Transport(nr), dom, per)
        assert np.array_equal(_flat(sfa), z["sum_out"]), f
        dboxes = [A.Box(r[:dim].tolist(), r[dim:].tolist()) for r in z["dst_boxes"]]
        dba = A.BoxArray(dboxes)
        dfa = A.MultiFab(dba, A.sfc_distribute(dba, A.default_costs(dba), nr), nc, 1)
        dfa.setval(0.0)
        A.parallel_copy(dfa, fa, A.Transport(nr), dom, per)
        assert np.array_equal(_flat(dfa), z["copy_out"]), f


def test_reference_golden_interlevel():
    z = np.load(os.path.join(GOLDEN, "interlevel.npz"))
    fba = A.BoxArray([A.Box(r[:3].tolist(), r[3:].tolist()) for r in z["fine_boxes"]])
    cba = A.BoxArray([A.Box(r[:3].tolist(), r[3:].tolist()) for r in z["crse_boxes"]])
    fine = A.MultiFab(fba, A.DistributionMapping.single_rank(2), 1, 0)
    crse = A.MultiFab(cba, A.DistributionMapping.single_rank(1), 1, 1)
    fine.fab(0).data.copy_(torch.as_tensor(z["fine_in0"]))
    fine.fab(1).data.copy_(torch.as_tensor(z["fine_in1"]))
    crse.setval(-3.0)
    A.average_down(fine, crse, 2, A.Transport(1))
    assert np.array_equal(crse.fab(0).data.cpu().numpy(), z["avg_out"])
    crse.fab(0).data.copy_(torch.as_tensor(z["crse_in"]))
    A.interp_to_fine(fine, crse, 2, A.Transport(1), method="pc")
    assert np.array_equal(fine.fab(0).data.cpu().numpy(), z["interp_out0"])
    assert np.array_equal(fine.fab(1).data.cpu().numpy(), z["interp_out1"])


def test_reference_golden_domain_bc():
    z = np.load(os.path.join(GOLDEN, "domain_bc.npz"))
    geom = A.Geometry(A.Box((0, 0), (7, 9)), (0.0, 0.0), (1.0, 1.0), False)
    ba = A.BoxArray([A.Box(r[:2].tolist(), r[2:].tolist()) for r in z["boxes"]])
    fa = A.MultiFab(ba, A.DistributionMapping.single_rank(2), 1, 2)
    fa.fab(0).data.copy_(torch.as_tensor(z["in0"]))
    fa.fab(1).data.copy_(torch.as_tensor(z["in1"]))
    rec = A.BoundaryRecord(("external", "extrap"), ("extrap", "external"), external_value=-1.5)
    A.apply_domain_boundary(fa, geom, rec)
    assert np.array_equal(fa.fab(0).data.cpu().numpy(), z["out0"])
    assert np.array_equal(fa.fab(1).data.cpu().numpy(), z["out1"])


def test_average_down_and_interp_match_oracle_3d(rng):
    dom = A.Box((0, 0, 0), (31, 31, 31))
    fba = A.BoxArray([dom]).max_size(16)
    cba = A.coarsened_layout(fba, 2)
    fine = A.MultiFab(fba, A.DistributionMapping.single_rank(len(fba)), 2, 1)
    crse = A.MultiFab(cba, A.DistributionMapping.single_rank(len(cba)), 2, 0)
    ff = M.make_fabs(tboxes(fba), 2, 1)
    for f in ff.values():
        f[...] = rng.normal(size=f.shape)
    load_device_from_oracle(fine, ff)
    cf = M.make_fabs(tboxes(cba), 2, 0)
    M.average_down(tboxes(fba), ff, 1, tboxes(cba), cf, 0, (2, 2, 2))
    A.average_down(fine, crse, 2, A.Transport(1))
    got = oracle_fabs_from_device(crse)
    for i in cf:
        assert np.array_equal(got[i], cf[i])
    # prolong-add onto a single-box coarse layout (agglomerated path)
    single = A.MultiFab(A.BoxArray([dom.coarsen(2)]), A.DistributionMapping.single_rank(1), 2, 0)
    sf = M.make_fabs([tbox_ for tbox_ in tboxes(single.ba)], 2, 0)
    sf[0][...] = rng.normal(size=sf[0].shape)
    load_device_from_oracle(single, sf)
    M.interp_pc(tboxes(fba), ff, 1, tboxes(single.ba), sf, 0, (2, 2, 2), add=True)
    A.interp_to_fine(fine, single, 2, A.Transport(1), add=True)
    got = oracle_fabs_from_device(fine)
    for i in ff:
        assert np.array_equal(got[i], ff[i])


def test_host_image_round_trip():
    """FabArray.to_host_image / from_host_image: comp-major per-box records of
    the resident boxes, one copy + one launch each way."""
    dom = A.Box((0, 0, 0), (47, 31, 15))
    ba = A.BoxArray([dom]).max_size(16)
    dm = A.DistributionMapping.single_rank(len(ba))
    src = A.MultiFab(ba, dm, 2, 1)
    src.storage.normal_()
    img = torch.empty(src.image_size(), dtype=torch.float64).pin_memory()
    src.to_host_image(img)
    torch.cuda.synchronize()
    off = 0
    for i in range(len(ba)):
        want = src.fab(i).valid().cpu().numpy().ravel()
        assert np.array_equal(img[off : off + want.size].numpy(), want)
        off += want.size
    dst = A.MultiFab(ba, dm, 2, 2)
    dst.from_host_image(img)
    torch.cuda.synchronize()
    for i in range(len(ba)):
        assert torch.equal(dst.fab(i).valid(), src.fab(i).valid())
