"""CPU: the ghost push / pull tables (ghosts.py) -- the 27 addresses per box
the streaming sweep stores through (push) or copies from (pull) -- emulated on
the host storage: both must leave every ghost cell within the width exactly
as FillBoundary defines it (fabarray.py:364-374: the periodic image's valid
value, boundary ghosts untouched)."""

import itertools

import numpy as np
import pytest

import paper_2009_12009_b200 as A
from paper_2009_12009_b200.ghosts import pull_table, push_table

DIRS = [d for d in itertools.product((-1, 0, 1), repeat=3) if d != (0, 0, 0)]
SENT = -7777.0


def _setup(shape, m, per, ngrow, seed):
    dom = A.Box((0, 0, 0), tuple(s - 1 for s in shape))
    ba = A.BoxArray([dom]).max_size(m)
    dm = A.DistributionMapping.single_rank(len(ba))
    fa = A.MultiFab(ba, dm, 1, ngrow)
    assert fa.storage.device.type == "cpu"
    g = np.random.default_rng(seed).standard_normal(shape)
    # host-side setup (the library's setval / load are CUDA-only by design)
    st = fa.storage.numpy()
    st[:] = SENT
    w = ngrow
    for i, fab in fa.fabs.items():
        B = ba[i]
        view = fab.data.numpy()
        view[0, w:view.shape[1] - w, w:view.shape[2] - w, w:view.shape[3] - w] = g[
            B.lo[0]:B.hi[0] + 1, B.lo[1]:B.hi[1] + 1, B.lo[2]:B.hi[2] + 1]
    return dom, ba, fa, g


def _geometry(fa):
    tab = fa.fabtab
    s0, s1, gw = int(tab[0][2]), int(tab[0][3]), fa.ngrow
    origin = [int(tab[b][0]) + gw * s0 + gw * s1 + gw for b in range(len(fa.ba))]
    return s0, s1, origin


def _expect(fa, b, dom, g, per, width):
    """Dense FillBoundary expectation for box b's grown region (width)."""
    B = fa.ba[b]
    ext = [B.hi[a] - B.lo[a] + 1 for a in range(3)]
    out = {}
    for i in range(-width, ext[0] + width):
        for j in range(-width, ext[1] + width):
            for k in range(-width, ext[2] + width):
                loc = (i, j, k)
                if all(0 <= loc[a] < ext[a] for a in range(3)):
                    continue
                p = [B.lo[a] + loc[a] for a in range(3)]
                ok = True
                for a in range(3):
                    n = dom.hi[a] - dom.lo[a] + 1
                    if not dom.lo[a] <= p[a] <= dom.hi[a]:
                        if per[a]:
                            p[a] = dom.lo[a] + (p[a] - dom.lo[a]) % n
                        else:
                            ok = False
                out[loc] = g[tuple(p)] if ok else SENT
    return out


def _check(fa, st, dom, g, per, width):
    s0, s1, origin = _geometry(fa)
    for b in range(len(fa.ba)):
        for loc, want in _expect(fa, b, dom, g, per, width).items():
            got = st[origin[b] + loc[0] * s0 + loc[1] * s1 + loc[2]]
            assert got == want, (b, loc, got, want)


CASES = [((16, 16, 16), 8, (True, True, True), 2, 2), ((16, 8, 12), 4, (True, False, True), 2, 2),
         ((12, 12, 12), 6, (False, False, False), 2, 1), ((16, 16, 8), 8, (True, True, False), 3, 3)]


@pytest.mark.parametrize("shape,m,per,ngrow,width", CASES)
def test_pull_table_emulated_equals_fill(shape, m, per, ngrow, width):
    dom, ba, fa, g = _setup(shape, m, per, ngrow, 1)
    tab = pull_table(fa, dom, per, width)
    assert tab is not None and not tab.remote
    st = fa.storage.numpy()
    src = st.copy()
    base = fa.storage.data_ptr()
    s0, s1, origin = _geometry(fa)
    for b in range(len(ba)):
        B = ba[b]
        ext = [B.hi[a] - B.lo[a] + 1 for a in range(3)]
        for d in DIRS:
            e = int(tab.host[b, (d[0] + 1) * 9 + (d[1] + 1) * 3 + (d[2] + 1)])
            if not e:
                continue
            q = ((e & ~1) - base) // 8
            rng = [range(-width, 0) if d[a] < 0 else (range(ext[a], ext[a] + width) if d[a] > 0 else range(ext[a]))
                   for a in range(3)]
            for i, j, k in itertools.product(*rng):
                st[origin[b] + i * s0 + j * s1 + k] = src[q + i * s0 + j * s1 + k]
    _check(fa, st, dom, g, per, width)


@pytest.mark.parametrize("shape,m,per,ngrow,width", CASES)
def test_push_table_emulated_equals_fill(shape, m, per, ngrow, width):
    dom, ba, fa, g = _setup(shape, m, per, ngrow, 2)
    tab = push_table(fa, dom, per, width)
    assert tab is not None and not tab.remote
    st = fa.storage.numpy()
    base = fa.storage.data_ptr()
    s0, s1, origin = _geometry(fa)
    for b in range(len(ba)):
        B = ba[b]
        ext = [B.hi[a] - B.lo[a] + 1 for a in range(3)]
        for d in DIRS:
            e = int(tab.host[b, (d[0] + 1) * 9 + (d[1] + 1) * 3 + (d[2] + 1)])
            if not e:
                continue
            q = (e - base) // 8
            rng = [range(width) if d[a] < 0 else (range(ext[a] - width, ext[a]) if d[a] > 0 else range(ext[a]))
                   for a in range(3)]
            for i, j, k in itertools.product(*rng):
                st[q + i * s0 + j * s1 + k] = st[origin[b] + i * s0 + j * s1 + k]
    _check(fa, st, dom, g, per, width)


def test_tables_reject_non_lattice_layouts():
    ba = A.BoxArray([A.Box((0, 0, 0), (15, 15, 7)), A.Box((0, 0, 8), (7, 15, 15)), A.Box((8, 0, 8), (15, 15, 15))])
    dm = A.DistributionMapping.single_rank(len(ba))
    f = A.MultiFab(ba, dm, 1, 2)
    dom = A.Box((0, 0, 0), (15, 15, 15))
    assert push_table(f, dom, True, 2) is None
    assert pull_table(f, dom, True, 2) is None
