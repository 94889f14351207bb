"""k_gsrb_stream (csrc/gsrb_stream.cu): the register-streamed fused GSRB sweep.

Checked bit for bit against the oracle's fill / red / fill / black
(oracle/mlmg_ref.py) and against the previous TMA sweep kernels
(library option "sweep_kernel" = 1) on the same inputs: periodic and
non-periodic (fixed ring cells), odd global box origins, many boxes, the
single big box the solver uses (several segments, alternating stream
directions), the fused prolongation (PROL) and the fused input-residual norm
(NORM) variants.
"""

import numpy as np
import pytest
import torch

import paper_2009_12009_b200 as A
from paper_2009_12009_b200 import stencil as S
from paper_2009_12009_b200._native import option
from paper_2009_12009_b200.interlevel import prolong_from
from oracle import mesh_ref as M
from oracle import mlmg_ref as R
from helpers import tboxes

pytestmark = pytest.mark.gpu

DH = (65536.0, 16384.0, 4096.0)


def _setup(rng, n, m, lo=0, periodic=True, shape=None):
    shape = shape or (n, n, n)
    dom = A.Box([lo] * 3, [lo + s - 1 for s in shape])
    ba = A.BoxArray([dom]).max_size(m)
    dm = A.DistributionMapping.single_rank(len(ba))
    tr = A.Transport(1)
    per = (periodic,) * 3
    a = A.MultiFab(ba, dm, 1, 2)
    rhs = A.MultiFab(ba, dm, 1, 1)
    g = rng.normal(size=(1,) + shape)
    gr = rng.normal(size=(1,) + shape)
    a.load_valid_from(dom, g)
    rhs.load_valid_from(dom, gr)
    A.fill_boundary(rhs, tr, dom, per)
    A.fill_boundary(a, tr, dom, per)
    return dom, ba, dm, tr, per, a, rhs, g, gr


def _valid(fa):
    return {i: f.valid().cpu().numpy().copy() for i, f in fa.fabs.items()}


def _sweep(a, rhs, fixed=None, legacy=False):
    b = A.MultiFab(a.ba, a.dm, 1, 2)
    with option("sweep_kernel", 1 if legacy else 0):
        S.gsrb_sweep(a, b, rhs, DH, fixed=fixed)
    torch.cuda.synchronize()
    return _valid(b)


def _eq(x, y):
    assert x.keys() == y.keys()
    for i in x:
        assert np.array_equal(x[i], y[i]), i


@pytest.mark.parametrize("n,m,lo", [(64, 64, 0), (128, 64, 0), (64, 64, 3), (128, 128, -7), (64, 32, 0), (96, 32, 5)])
def test_stream_sweep_matches_oracle_and_legacy(rng, n, m, lo):
    dom, ba, dm, tr, per, a, rhs, g, gr = _setup(rng, n, m, lo)
    got = _sweep(a, rhs)
    _eq(got, _sweep(a, rhs, legacy=True))
    boxes = tboxes(ba)
    d = (tuple(dom.lo), tuple(dom.hi))
    pf = M.make_fabs(boxes, 1, 1)
    rf = M.make_fabs(boxes, 1, 0)
    M.load_global(boxes, pf, 1, d, g)
    M.load_global(boxes, rf, 0, d, gr)
    for color in (0, 1):
        M.fill_boundary(boxes, pf, 1, d, per)
        for i, bx in enumerate(boxes):
            R.gsrb_color(bx, pf[i][0], rf[i][0], DH, color)
    for i in got:
        assert np.array_equal(got[i], M.valid(boxes, pf, 1, i)), i


@pytest.mark.parametrize("shape", [(256, 256, 256), (96, 64, 128), (6, 64, 64)])
def test_stream_segments_and_directions(rng, shape):
    """One big box: the column is cut into several plane segments streamed in
    alternating directions (and a box too thin for more than one segment)."""
    dom, ba, dm, tr, per, a, rhs, g, gr = _setup(rng, 0, 256, shape=shape)
    _eq(_sweep(a, rhs), _sweep(a, rhs, legacy=True))


@pytest.mark.parametrize("lo", [0, 5])
def test_stream_fixed_ring(rng, lo):
    """Non-periodic domain: ring cells outside it are never relaxed (they keep
    their ghost values); cells inside it are recomputed as by the owner."""
    dom, ba, dm, tr, per, a, rhs, g, gr = _setup(rng, 128, 64, lo, periodic=False)
    # arbitrary values in the out-of-domain ghosts (a boundary condition)
    for f in a.fabs.values():
        v = f.data
        mask = torch.ones_like(v, dtype=torch.bool)
        mask[(slice(None),) + tuple(slice(2, -2) for _ in range(3))] = False
        v[mask] = torch.randn(int(mask.sum()), dtype=torch.float64, device=v.device)
    A.fill_boundary(a, tr, dom, per)
    _eq(_sweep(a, rhs, fixed=dom), _sweep(a, rhs, fixed=dom, legacy=True))
    # a partly fixed box: unbounded in i, fixed in j and k
    fx = ((None, dom.lo[1], dom.lo[2]), (None, dom.hi[1], dom.hi[2]))
    _eq(_sweep(a, rhs, fixed=fx), _sweep(a, rhs, fixed=fx, legacy=True))


@pytest.mark.parametrize("n,m", [(128, 64), (256, 256)])
def test_stream_prolong_fused(rng, n, m):
    """PROL: b = sweep(a + pc(c)) == prolong(add); fill(2); sweep -- bitwise
    (the reference composition runs the other sweep kernels)."""
    dom, ba, dm, tr, per, a, rhs, g, gr = _setup(rng, n, m)
    cba = A.coarsened_layout(ba, 2)
    cdom = dom.coarsen(2)
    c = A.MultiFab(cba, dm, 1, 1)
    c.load_valid_from(cdom, rng.normal(size=(1,) + tuple(cdom.extents())))
    A.fill_boundary(c, tr, cdom, per)
    out = {}
    b = A.MultiFab(ba, dm, 1, 2)
    S.gsrb_sweep_prolong(a, b, rhs, DH, c)
    torch.cuda.synchronize()
    out[False] = _valid(b)
    a2 = A.MultiFab(ba, dm, 1, 2)
    a2.storage.copy_(a.storage)
    prolong_from(a2, c, (2, 2, 2), add=True)
    A.fill_boundary(a2, tr, dom, per)
    _eq(out[False], _sweep(a2, rhs, legacy=True))


@pytest.mark.parametrize("n,m", [(64, 64), (256, 256), (128, 64)])
def test_stream_norm(rng, n, m):
    """NORM: the sweep output is unchanged and the fused max |rhs - L(a)| equals
    the residual-norm kernel on a, bit for bit."""
    dom, ba, dm, tr, per, a, rhs, g, gr = _setup(rng, n, m)
    b = A.MultiFab(ba, dm, 1, 2)
    nrm = torch.zeros(1, dtype=torch.int64, device="cuda")
    S.gsrb_sweep_norm(a, b, rhs, DH, nrm)
    torch.cuda.synchronize()
    _eq(_valid(b), _sweep(a, rhs))
    fused = nrm.view(torch.float64).item()
    r = A.MultiFab(ba, dm, 1, 0)
    S.residual(r, rhs, a, DH)
    ref = A.device_reduce(r, "absmax").item()
    assert fused == ref and fused > 0


def test_stream_norm_nan_propagates(rng):
    dom, ba, dm, tr, per, a, rhs, g, gr = _setup(rng, 64, 64)
    a.fab(0).data[0, 10, 11, 12] = float("nan")
    b = A.MultiFab(ba, dm, 1, 2)
    nrm = torch.zeros(1, dtype=torch.int64, device="cuda")
    S.gsrb_sweep_norm(a, b, rhs, DH, nrm)
    assert np.isnan(nrm.view(torch.float64).item())


def test_stream_not_applicable_raises_for_norm(rng):
    """16-wide boxes do not take the streaming path: the plain sweep falls back
    to the other kernels, the norm variant raises NotImplementedError."""
    dom, ba, dm, tr, per, a, rhs, g, gr = _setup(rng, 64, 16)
    b = A.MultiFab(ba, dm, 1, 2)
    nrm = torch.zeros(1, dtype=torch.int64, device="cuda")
    with pytest.raises(NotImplementedError):
        S.gsrb_sweep_norm(a, b, rhs, DH, nrm)


@pytest.mark.parametrize("cfg", [1, 2, 4, 6])
def test_stream_variants_agree(rng, cfg):
    """Every compiled tile / strip / depth variant (library option
    "stream_config") gives the same bits for the plain, PROL and NORM sweeps."""
    dom, ba, dm, tr, per, a, rhs, g, gr = _setup(rng, 128, 128)
    cba = A.coarsened_layout(ba, 2)
    cdom = dom.coarsen(2)
    c = A.MultiFab(cba, dm, 1, 1)
    c.load_valid_from(cdom, rng.normal(size=(1,) + tuple(cdom.extents())))
    A.fill_boundary(c, tr, cdom, per)
    want_plain = _sweep(a, rhs, legacy=True)
    a2 = A.MultiFab(ba, dm, 1, 2)
    a2.storage.copy_(a.storage)
    prolong_from(a2, c, (2, 2, 2), add=True)
    A.fill_boundary(a2, tr, dom, per)
    want_prol = _sweep(a2, rhs, legacy=True)
    r = A.MultiFab(ba, dm, 1, 0)
    S.residual(r, rhs, a, DH)
    want_norm = A.device_reduce(r, "absmax").item()
    with option("stream_config", cfg):
        _eq(_sweep(a, rhs), want_plain)
        b = A.MultiFab(ba, dm, 1, 2)
        S.gsrb_sweep_prolong(a, b, rhs, DH, c)
        torch.cuda.synchronize()
        _eq(_valid(b), want_prol)
        nrm = torch.zeros(1, dtype=torch.int64, device="cuda")
        b = A.MultiFab(ba, dm, 1, 2)
        S.gsrb_sweep_norm(a, b, rhs, DH, nrm)
        torch.cuda.synchronize()
        _eq(_valid(b), want_plain)
        assert nrm.view(torch.float64).item() == want_norm


@pytest.mark.parametrize("n,m,per", [(64, 32, True), (128, 64, True), (64, 64, True), (128, 128, True),
                                     (128, 64, False), (96, 32, True)])
def test_push_equals_fill(rng, n, m, per):
    """Ghost push (ghosts.push_table): the sweep, its NORM variant and the
    fused prolongation sweep leave every cell of every grown box -- valid and
    ghost -- exactly as the same kernel followed by fill_boundary(width 2)."""
    from paper_2009_12009_b200.ghosts import push_table

    dom, ba, dm, tr, p3, a, rhs, g, gr = _setup(rng, n, m, periodic=per)
    fixed = None if per else dom
    cba = A.coarsened_layout(ba, 2)
    cdom = dom.coarsen(2)
    c = A.MultiFab(cba, dm, 1, 1)
    c.load_valid_from(cdom, rng.normal(size=(1,) + tuple(cdom.extents())))
    A.fill_boundary(c, tr, cdom, p3)
    runs = [("sweep", lambda b, t: S.gsrb_sweep(a, b, rhs, DH, fixed=fixed, push=t)),
            ("norm", lambda b, t: S.gsrb_sweep_norm(a, b, rhs, DH, torch.zeros(1, dtype=torch.int64, device="cuda"),
                                                    fixed=fixed, push=t))]
    if per:
        runs.append(("prolong", lambda b, t: S.gsrb_sweep_prolong(a, b, rhs, DH, c, push=t)))
    for name, fn in runs:
        b1 = A.MultiFab(ba, dm, 1, 2)
        b2 = A.MultiFab(ba, dm, 1, 2)
        fn(b1, None)
        A.fill_boundary(b1, tr, dom, p3, ngrow=2)
        tab = push_table(b2, dom, p3, 2)
        assert tab is not None and not tab.remote
        fn(b2, tab)
        torch.cuda.synchronize()
        for i in b1.fabs:
            assert torch.equal(b1.fab(i).data, b2.fab(i).data), (name, i)


@pytest.mark.parametrize("n,m", [(64, 32), (128, 64), (64, 64), (96, 32)])
def test_pull_equals_fill(rng, n, m):
    """Ghost pull (ghosts.pull_table): the sweep and its NORM variant, run on
    an input whose ghosts hold garbage, produce the bits of fill_boundary(width
    2) + the sweep, and leave the input's ghosts exactly as that fill does."""
    from paper_2009_12009_b200.ghosts import pull_table

    dom, ba, dm, tr, p3, a, rhs, g, gr = _setup(rng, n, m)
    for name in ("sweep", "norm"):
        ref_b = A.MultiFab(ba, dm, 1, 2)
        n1 = torch.zeros(1, dtype=torch.int64, device="cuda")
        if name == "sweep":
            S.gsrb_sweep(a, ref_b, rhs, DH)
        else:
            S.gsrb_sweep_norm(a, ref_b, rhs, DH, n1)
        a2 = A.MultiFab(ba, dm, 1, 2)
        a2.setval(-7777.0)
        a2.load_valid_from(dom, g)
        tab = pull_table(a2, dom, p3, 2)
        assert tab is not None and not tab.remote
        b2 = A.MultiFab(ba, dm, 1, 2)
        n2 = torch.zeros(1, dtype=torch.int64, device="cuda")
        S.gsrb_sweep_pull(a2, b2, rhs, DH, tab, norm=None if name == "sweep" else n2)
        torch.cuda.synchronize()
        _eq(_valid(ref_b), _valid(b2))
        for i in a.fabs:
            assert torch.equal(a.fab(i).data, a2.fab(i).data), (name, i)
        assert torch.equal(n1, n2), name


def test_pull_table_rejects_irregular_layout():
    from paper_2009_12009_b200.ghosts import pull_table

    ba = A.BoxArray([A.Box((0, 0, 0), (63, 63, 31)), A.Box((0, 0, 32), (31, 63, 63)), A.Box((32, 0, 32), (63, 63, 63))])
    dm = A.DistributionMapping.single_rank(len(ba))
    f = A.MultiFab(ba, dm, 1, 2)
    assert pull_table(f, A.Box((0, 0, 0), (63, 63, 63)), True, 2) is None


def test_push_table_rejects_irregular_layout():
    from paper_2009_12009_b200.ghosts import push_table

    ba = A.BoxArray([A.Box((0, 0, 0), (63, 63, 31)), A.Box((0, 0, 32), (31, 63, 63)), A.Box((32, 0, 32), (63, 63, 63))])
    dm = A.DistributionMapping.single_rank(len(ba))
    f = A.MultiFab(ba, dm, 1, 2)
    assert push_table(f, A.Box((0, 0, 0), (63, 63, 63)), True, 2) is None


@pytest.mark.parametrize("shape,m", [((256, 256, 256), 256), ((128, 128, 128), 64), ((64, 64, 64), 32),
                                     ((96, 64, 128), 128), ((6, 32, 64), 64)])
def test_stream_resid_restrict(rng, shape, m):
    """k_resid_restrict_stream == the tile kernel (k_resid_restrict, sweep_kernel
    option 1) == the oracle's residual + average_down, bit for bit; several
    plane segments per column, streamed both ways."""
    dom, ba, dm, tr, per, a, rhs, g, gr = _setup(rng, 0, m, shape=shape)
    cba = A.coarsened_layout(ba, 2)
    out = {}
    for legacy in (False, True):
        c = A.MultiFab(cba, dm, 1, 1)
        with option("sweep_kernel", 1 if legacy else 0):
            S.residual_restrict(c, rhs, a, DH)
        torch.cuda.synchronize()
        out[legacy] = _valid(c)
    _eq(out[False], out[True])
    if shape[0] * shape[1] * shape[2] <= 64**3:
        boxes = tboxes(ba)
        d = (tuple(dom.lo), tuple(dom.hi))
        pf = M.make_fabs(boxes, 1, 1)
        rf = M.make_fabs(boxes, 1, 0)
        M.load_global(boxes, pf, 1, d, g)
        M.load_global(boxes, rf, 0, d, gr)
        M.fill_boundary(boxes, pf, 1, d, per)
        r = {i: (rf[i][0] - R.laplacian(pf[i][0], DH))[None] for i in pf}
        cf = M.make_fabs(tboxes(cba), 1, 0)
        M.average_down(boxes, r, 0, tboxes(cba), cf, 0, (2, 2, 2))
        for i in cf:
            assert np.array_equal(out[False][i], cf[i]), i
