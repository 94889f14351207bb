"""Device stencil kernels vs the oracle (bit-exact: the library is built with
--fmad=false and every kernel keeps the oracle's operand order)."""

import numpy as np
import pytest
import torch

import paper_2009_12009_b200 as A
from paper_2009_12009_b200 import stencil as S
from oracle import mesh_ref as M
from oracle import mlmg_ref as R
from helpers import load_device_from_oracle, oracle_fabs_from_device, tboxes

pytestmark = pytest.mark.gpu


def _layout(n, m, lo=0):
    dom = A.Box([lo] * 3, [lo + n - 1] * 3)
    ba = A.BoxArray([dom]).max_size(m)
    return dom, ba, A.DistributionMapping.single_rank(len(ba))


def _random_fabs(rng, ba, ng):
    f = M.make_fabs(tboxes(ba), 1, ng)
    for a in f.values():
        a[...] = rng.normal(size=a.shape)
    return f


DH = (65536.0, 16384.0, 4096.0)


@pytest.mark.parametrize("n,m,lo", [(16, 8, 0), (32, 16, -7), (24, 12, 3), (64, 32, 0)])
def test_laplacian_and_residual_bitexact(rng, n, m, lo):
    dom, ba, dm = _layout(n, m, lo)
    phi = A.MultiFab(ba, dm, 1, 1)
    rhs = A.MultiFab(ba, dm, 1, 0)
    out = A.MultiFab(ba, dm, 1, 0)
    pf = _random_fabs(rng, ba, 1)
    rf = _random_fabs(rng, ba, 0)
    load_device_from_oracle(phi, pf)
    load_device_from_oracle(rhs, rf)
    S.laplacian(out, phi, DH)
    got = oracle_fabs_from_device(out)
    for i in pf:
        assert np.array_equal(got[i][0], R.laplacian(pf[i][0], DH))
    S.residual(out, rhs, phi, DH)
    got = oracle_fabs_from_device(out)
    for i in pf:
        assert np.array_equal(got[i][0], rf[i][0] - R.laplacian(pf[i][0], DH))


@pytest.mark.parametrize("n,m,lo", [(16, 8, 0), (20, 10, -3), (64, 32, 1)])
def test_gsrb_color_bitexact(rng, n, m, lo):
    dom, ba, dm = _layout(n, m, lo)
    phi = A.MultiFab(ba, dm, 1, 1)
    rhs = A.MultiFab(ba, dm, 1, 0)
    pf = _random_fabs(rng, ba, 1)
    rf = _random_fabs(rng, ba, 0)
    load_device_from_oracle(phi, pf)
    load_device_from_oracle(rhs, rf)
    boxes = tboxes(ba)
    for color in (0, 1):
        S.gsrb_color(phi, rhs, DH, color)
        for i, b in enumerate(boxes):
            R.gsrb_color(b, pf[i][0], rf[i][0], DH, color)
        got = oracle_fabs_from_device(phi)
        for i in pf:
            assert np.array_equal(got[i], pf[i])


@pytest.mark.parametrize("n,m", [(16, 8), (32, 16), (64, 32), (128, 64), (8, 4), (8, 8), (12, 6), (40, 20)])
def test_fused_sweep_equals_fill_red_fill_black(rng, n, m):
    dom, ba, dm = _layout(n, m)
    tr = A.Transport(1)
    per = (True,) * 3
    a = A.MultiFab(ba, dm, 1, 2)
    b = A.MultiFab(ba, dm, 1, 2)
    rhs = A.MultiFab(ba, dm, 1, 1)
    g = rng.normal(size=(1, n, n, n))
    gr = rng.normal(size=(1, n, n, n))
    a.load_valid_from(dom, g)
    rhs.load_valid_from(dom, gr)
    A.fill_boundary(rhs, tr, dom, per)
    boxes = tboxes(ba)
    d = (tuple(dom.lo), tuple(dom.hi))
    pf = M.make_fabs(boxes, 1, 1)
    rf = M.make_fabs(boxes, 1, 0)
    M.load_global(boxes, pf, 1, d, g)
    M.load_global(boxes, rf, 0, d, gr)
    for sweep in range(3):
        A.fill_boundary(a, tr, dom, per)
        S.gsrb_sweep(a, b, rhs, DH)
        a, b = b, a
        for color in (0, 1):
            M.fill_boundary(boxes, pf, 1, d, per)
            for i, bx in enumerate(boxes):
                R.gsrb_color(bx, pf[i][0], rf[i][0], DH, color)
        got = oracle_fabs_from_device(a)
        for i in pf:
            want = M.valid(boxes, pf, 1, i)
            have = got[i][(slice(None),) + M.region_index(boxes[i], 2, boxes[i])]
            assert np.array_equal(have, want), (sweep, i)


def test_residual_restrict_bitexact(rng):
    dom, ba, dm = _layout(32, 16)
    cba = A.coarsened_layout(ba, 2)
    phi = A.MultiFab(ba, dm, 1, 1)
    rhs = A.MultiFab(ba, dm, 1, 1)
    crse = A.MultiFab(cba, dm, 1, 1)
    pf = _random_fabs(rng, ba, 1)
    rf = _random_fabs(rng, ba, 1)
    load_device_from_oracle(phi, pf)
    load_device_from_oracle(rhs, rf)
    S.residual_restrict(crse, rhs, phi, DH)
    boxes = tboxes(ba)
    r = {i: (M.valid(boxes, rf, 1, i)[0] - R.laplacian(pf[i][0], DH))[None] for i in pf}
    cf = M.make_fabs(tboxes(cba), 1, 1)
    M.average_down(boxes, r, 0, tboxes(cba), cf, 1, (2, 2, 2))
    got = oracle_fabs_from_device(crse)
    for i in cf:
        sl = (slice(None),) + M.region_index(tboxes(cba)[i], 1, tboxes(cba)[i])
        assert np.array_equal(got[i][sl], cf[i][sl])


@pytest.mark.parametrize("n,m,lo", [(128, 128, 0), (128, 64, 0), (64, 32, 0), (64, 64, -32)])
def test_sweep_prolong_equals_prolong_fill_sweep(n, m, lo):
    """k_gsrb_sweep5<PROL>: GSRB(a + pc(c)) == prolong_from(add); fill(2);
    gsrb_sweep, bit for bit on every valid cell; `a` is left unchanged."""
    from paper_2009_12009_b200.interlevel import coarsened_layout, prolong_from

    dom, ba, dm = _layout(n, m, lo)
    tr = A.Transport(1)
    g = torch.Generator(device="cuda").manual_seed(11)

    def rnd(fa):
        fa.storage.copy_(torch.randn(fa.storage.shape, generator=g, device="cuda", dtype=torch.float64))

    a = A.MultiFab(ba, dm, 1, 2)
    rhs = A.MultiFab(ba, dm, 1, 1)
    rnd(a)
    rnd(rhs)
    cba = coarsened_layout(ba, 2)
    c = A.MultiFab(cba, dm, 1, 2)
    rnd(c)
    A.fill_boundary(a, tr, dom, True, ngrow=2)
    A.fill_boundary(rhs, tr, dom, True)
    A.fill_boundary(c, tr, dom.coarsen(2), True, ngrow=1)
    a0 = a.storage.clone()
    dh = (float(n * n), 0.5 * n * n, 2.0 * n * n)
    fused = A.MultiFab(ba, dm, 1, 2)
    S.gsrb_sweep_prolong(a, fused, rhs, dh, c)
    assert torch.equal(a.storage, a0)  # the input is not modified
    ref = A.MultiFab(ba, dm, 1, 2)
    prolong_from(a, c, (2, 2, 2), add=True)
    A.fill_boundary(a, tr, dom, True, ngrow=2)
    S.gsrb_sweep(a, ref, rhs, dh)
    torch.cuda.synchronize()
    for i in ref.fabs:
        assert torch.equal(ref.fab(i).valid(), fused.fab(i).valid()), i


def test_sweep_prolong_rejects_non_coarsened_layout():
    dom, ba, dm = _layout(64, 32)
    a = A.MultiFab(ba, dm, 1, 2)
    rhs = A.MultiFab(ba, dm, 1, 1)
    b = A.MultiFab(ba, dm, 1, 2)
    # same box count, but the "coarse" boxes are shifted by one cell: not the
    # coarsened fine boxes
    wrong = A.MultiFab(A.BoxArray([A.Box((1, 0, 0), (32, 31, 31))]).max_size(16), dm, 1, 1)
    assert len(wrong.ba) == len(ba)
    with pytest.raises(ValueError):
        S.gsrb_sweep_prolong(a, b, rhs, (1.0, 1.0, 1.0), wrong)
