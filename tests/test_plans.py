"""Native (C++) plan builders vs the oracle restatement and the reference's
golden plan tables (CPU: plans are host code; no device call is made)."""

import glob
import os

import numpy as np
import pytest

import paper_2009_12009_b200 as A
from paper_2009_12009_b200 import counters
from oracle import mesh_ref as M
from helpers import random_cover, tboxes

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _layout(rng, dim):
    n = int(rng.integers(8, 24))
    dom = A.Box([0] * dim, [n - 1] * dim)
    return dom, random_cover(rng, dom, nsplits=int(rng.integers(2, 10)))


@pytest.mark.parametrize("dim", [1, 2, 3])
def test_fill_plan_matches_oracle(rng, dim):
    for _ in range(12):
        dom, ba = _layout(rng, dim)
        per = tuple(bool(rng.integers(0, 2)) for _ in range(dim))
        ng = int(rng.integers(1, 4))
        plan = A.build_plan_fill_boundary(ba, ng, dom, per)
        want = M.records_table(M.fill_records(tboxes(ba), ng, (tuple(dom.lo), tuple(dom.hi)), per))
        assert np.array_equal(plan.table(), want)


def test_fill_plan_records_objects(rng):
    dom, ba = _layout(rng, 3)
    plan = A.build_plan_fill_boundary(ba, 1, dom, True)
    keys = [r.sort_key() for r in plan.records]
    assert keys == sorted(keys)
    for r in plan.records:
        assert r.dst_box == r.src_box.shift(r.shift)


@pytest.mark.parametrize("dim", [2, 3])
def test_copy_and_sum_plans_match_oracle(rng, dim):
    for _ in range(8):
        dom, src = _layout(rng, dim)
        dst = random_cover(rng, dom, nsplits=5)
        per = tuple(bool(rng.integers(0, 2)) for _ in range(dim))
        d = (tuple(dom.lo), tuple(dom.hi))
        got = A.build_plan_copy(dst, src, dom, per).table()
        assert np.array_equal(got, M.records_table(M.copy_records(tboxes(dst), tboxes(src), 0, d, per)))
        got = A.build_plan_copy(dst, src).table()
        assert np.array_equal(got, M.records_table(M.copy_records(tboxes(dst), tboxes(src))))
        got = A.build_plan_copy_grown(dst, src, 1, dom, per).table()
        assert np.array_equal(got, M.records_table(M.copy_records(tboxes(dst), tboxes(src), 1, d, per)))
        got = A.build_plan_sum_boundary(src, 1, dom, per).table()
        assert np.array_equal(got, M.records_table(M.sum_records(tboxes(src), 1, d, per)))


def test_fill_plan_matches_reference_golden():
    files = sorted(glob.glob(os.path.join(GOLDEN, "mesh_case*.npz")))
    assert files, "golden fixtures missing"
    for f in files:
        z = np.load(f)
        dim = int(z["dim"])
        boxes = [A.Box(r[:dim].tolist(), r[dim:].tolist()) for r in z["boxes"]]
        dom = A.Box(z["domain"][:dim].tolist(), z["domain"][dim:].tolist())
        plan = A.build_plan_fill_boundary(A.BoxArray(boxes), int(z["ngrow"]), dom, tuple(bool(p) for p in z["periodic"]))
        assert np.array_equal(plan.table(), z["plan"]), f


def test_periodic_ghost_wider_than_domain_rejected():
    dom = A.Box((0, 0), (2, 2))
    with pytest.raises(ValueError):
        A.build_plan_fill_boundary(A.BoxArray([dom]), 4, dom, True)


def test_plan_cache_and_counter(rng):
    dom, ba = _layout(rng, 2)
    A.plan_cache_clear()
    counters.reset("plans_built")
    p1 = A.build_plan_fill_boundary(ba, 2, dom, (True, True))
    p2 = A.build_plan_fill_boundary(ba, 2, dom, (True, True))
    assert p1 is p2 and counters.get("plans_built") == 1
    A.build_plan_fill_boundary(ba, 1, dom, (True, True))
    assert counters.get("plans_built") == 2


def test_config_record_counts():
    """208 records for C1 periodic, 56 non-periodic; 106,496 for C5."""
    dom = A.Box((0, 0, 0), (63, 63, 63))
    ba = A.BoxArray([dom]).max_size(32)
    assert len(A.build_plan_fill_boundary(ba, 1, dom, True)) == 208
    assert len(A.build_plan_fill_boundary(ba, 1, dom, False)) == 56
    n, cells = A.build_plan_fill_boundary(ba, 1, dom, True).size()
    assert cells == 8 * (34**3 - 32**3)
    dom5 = A.Box((0, 0, 0), (511, 511, 511))
    ba5 = A.BoxArray([dom5]).max_size(32)
    n5, cells5 = A.build_plan_fill_boundary(ba5, 1, dom5, True).size()
    assert n5 == 106_496 and cells5 == 26_771_456


def test_plan_pairs(rng):
    dom, ba = _layout(rng, 2)
    dm = A.sfc_distribute(ba, A.default_costs(ba), 3)
    plan = A.build_plan_fill_boundary(ba, 1, dom, True)
    groups = plan.pairs(dm, dm)
    t = plan.table()
    for (s, d), rids in groups.items():
        assert rids == sorted(rids)
        for r in rids:
            assert dm[t[r, 0]] == s and dm[t[r, 1]] == d
    assert sum(len(v) for v in groups.values()) == len(plan)
