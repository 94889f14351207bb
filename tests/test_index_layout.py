"""Host metadata: box algebra, BoxArray hash, distribution (CPU).

Mirrors the reference's tests/test_index_space.py, test_boxarray.py,
test_distribution.py and acceptance criteria #1, #2, #4."""

import itertools

import numpy as np
import pytest

import paper_2009_12009_b200 as A
from paper_2009_12009_b200 import counters
from helpers import random_cover


def random_box(rng, dim, span=24, max_ext=8):
    lo = [int(rng.integers(-span, span)) for _ in range(dim)]
    e = [int(rng.integers(1, max_ext + 1)) for _ in range(dim)]
    return A.Box(lo, [l + x - 1 for l, x in zip(lo, e)])


def test_box_algebra_randomised(rng):
    for _ in range(2000):
        dim = int(rng.integers(1, 4))
        a, b, c = (random_box(rng, dim) for _ in range(3))
        ab = a.intersect(b)
        assert ab == b.intersect(a)
        assert ab.intersect(c) == a.intersect(b.intersect(c))
        if not ab.is_empty():
            assert a.contains_box(ab) and b.contains_box(ab)
        r = A.IntVect([int(rng.integers(2, 5))] * dim)
        assert a.refine(r).coarsen(r) == a
        assert a.coarsen(r).refine(r).contains_box(a)


def test_empty_box_normalisation_and_floor_coarsen():
    e = A.Box((3, 3), (1, 5))
    assert e.is_empty() and e == A.Box.empty(2)
    assert tuple(e.lo) == (0, 0) and tuple(e.hi) == (-1, 0)
    b = A.Box((-3, -1), (2, 4)).coarsen(2)
    assert tuple(b.lo) == (-2, -1) and tuple(b.hi) == (1, 2)


def test_box_diff_is_exact_partition(rng):
    for _ in range(300):
        dim = int(rng.integers(1, 4))
        a, b = random_box(rng, dim), random_box(rng, dim)
        pieces = A.box_diff(a, b)
        cells = set()
        for p in pieces:
            pc = set(p.cells())
            assert not (cells & pc)
            cells |= pc
        assert cells == set(a.cells()) - set(b.cells())


def test_box_diff_slab_order():
    v = A.Box((0, 0, 0), (3, 3, 3))
    pieces = A.box_diff(v.grow(1), v)
    # dimension 0 first, low slab then high slab (index_space.py:334-344)
    assert [tuple(p.lo) for p in pieces] == [
        (-1, -1, -1), (4, -1, -1), (0, -1, -1), (0, 4, -1), (0, 0, -1), (0, 0, 4)
    ]


def test_hash_matches_brute_force_and_bin_bound(rng):
    for _ in range(60):
        dim = int(rng.integers(2, 4))
        n = int(rng.integers(12, 28))
        dom = A.Box([0] * dim, [n - 1] * dim)
        ba = random_cover(rng, dom, nsplits=int(rng.integers(4, 8)))
        ba.intersections(ba[0])
        for _ in range(5):
            q = ba[int(rng.integers(len(ba)))].grow(1)
            before = counters.get("hash_bins_examined")
            got = sorted(ba.intersections(q), key=lambda t: t[0])
            assert counters.get("hash_bins_examined") - before <= 3**dim
            want = [(i, ba[i].intersect(q)) for i in range(len(ba)) if ba[i].intersects(q)]
            assert got == want


def test_boxarray_overlap_rejected():
    with pytest.raises(ValueError):
        A.BoxArray([A.Box((0, 0), (3, 3)), A.Box((3, 3), (5, 5))])


def test_max_size_chops_from_each_lo():
    ba = A.BoxArray([A.Box((0, 0, 0), (63, 63, 63))]).max_size(32)
    assert len(ba) == 8
    assert [tuple(b.lo) for b in ba][:3] == [(0, 0, 0), (0, 0, 32), (0, 32, 0)]
    ba = A.BoxArray([A.Box((0,), (9,))]).max_size(4)
    assert [(b.lo[0], b.hi[0]) for b in ba] == [(0, 3), (4, 7), (8, 9)]


def test_knapsack_known_answer():
    cost = [5, 4, 3, 3, 2, 1]
    dm = A.knapsack_distribute(cost, 3)
    assert A.load_stats(dm, cost)["max_load"] == 6.0


def test_sfc_contiguous_and_every_rank_gets_a_box():
    ba = A.BoxArray([A.Box((0, 0, 0), (255, 255, 255))]).max_size(64)
    for r in (1, 2, 4, 8):
        dm = A.sfc_distribute(ba, A.default_costs(ba), r)
        counts = np.bincount(dm.owner, minlength=r)
        assert counts.min() >= 1 and counts.sum() == 64
    dm8 = A.sfc_distribute(A.BoxArray([A.Box((0, 0, 0), (511, 511, 511))]).max_size(64), None or np.ones(512), 8)
    assert np.bincount(dm8.owner).tolist() == [64] * 8


def test_morton_key_interleave():
    dom = A.Box((0, 0, 0), (7, 7, 7))
    assert A.morton_key((1, 0, 0), dom) == 1
    assert A.morton_key((0, 1, 0), dom) == 2
    assert A.morton_key((0, 0, 1), dom) == 4
    assert A.morton_key((2, 0, 0), dom) == 8


def test_matches_reference_layout_layer(amrkit, rng):
    """Same chop, SFC map and knapsack as the reference (build container only)."""
    from amrkit.distribution import default_costs as rdc, knapsack_distribute as rks, sfc_distribute as rsfc

    for _ in range(30):
        dim = int(rng.integers(1, 4))
        n = int(rng.integers(16, 64))
        m = int(rng.integers(4, 17))
        rb = amrkit.BoxArray([amrkit.Box(amrkit.IntVect([0] * dim), amrkit.IntVect([n - 1] * dim))]).max_size(m)
        ob = A.BoxArray([A.Box([0] * dim, [n - 1] * dim)]).max_size(m)
        assert [(tuple(b.lo), tuple(b.hi)) for b in ob] == [(b.lo.coords, b.hi.coords) for b in rb]
        R = int(rng.integers(1, 9))
        assert A.sfc_distribute(ob, A.default_costs(ob), R).owner == rsfc(rb, rdc(rb), R).owner
        cost = rng.integers(1, 100, size=len(ob)).astype(float)
        assert A.knapsack_distribute(cost, R).owner == rks(cost, R).owner


def test_plotfile_header_text_matches_reference_golden():
    """The device writer's Header (pure host code) equals amrkit's, for the
    golden cases (tests/golden/plotfile.json, made from the reference)."""
    import json
    import os
    import sys
    import types

    import paper_2009_12009_b200 as A
    from paper_2009_12009_b200.plotfile import _header_text

    here = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
    sys.path.insert(0, here)
    import plotfile_cases as PC

    gold = json.load(open(os.path.join(here, "plotfile.json")))
    for name, dim, n, m, ncomp, nranks, two, time, names in PC.CASES:
        domain = A.Box(A.IntVect([0] * dim), A.IntVect([n - 1] * dim))
        g0 = A.Geometry(domain, (0.0,) * dim, (1.0,) * dim, (True,) * dim)
        levels = [(A.BoxArray([domain]).max_size(m), g0)]
        if two:
            fine = A.Box(A.IntVect([n // 2] * dim), A.IntVect([n + n // 2 - 1] * dim))
            levels.append((A.BoxArray([fine]).max_size(m), g0.refine(A.IntVect([2] * dim))))
        meshes = [types.SimpleNamespace(ba=ba, ncomp=ncomp) for ba, _ in levels]
        header = A.PlotfileHeader(time, names, [g for _, g in levels])
        assert _header_text(header, meshes) == gold[name]["header"]
