"""MLMG solve on the device vs the oracle V-cycle: same iteration count, same
residual history and bit-identical solution."""

import os

import numpy as np
import pytest
import torch

import paper_2009_12009_b200 as A
from oracle import mlmg_ref as R
from helpers import tboxes

pytestmark = pytest.mark.gpu


def _problem(n, m, seed):
    dom = A.Box((0, 0, 0), (n - 1,) * 3)
    ba = A.BoxArray([dom]).max_size(m)
    dm = A.DistributionMapping.single_rank(len(ba))
    geom = A.Geometry(dom, (0.0,) * 3, (1.0,) * 3, True)
    rng = np.random.default_rng(seed)
    rhs = rng.standard_normal((n, n, n))
    rhs -= rhs.mean()
    return dom, ba, dm, geom, rhs


def _solve_device(dom, ba, dm, geom, rhs, use_graph=True, nranks=1):
    if nranks > 1:
        dm = A.sfc_distribute(ba, A.default_costs(ba), nranks)
    phi = A.MultiFab(ba, dm, 1, 1)
    b = A.MultiFab(ba, dm, 1, 0)
    b.load_valid_from(dom, rhs)
    mg = A.MLMG(geom, ba, dm, transport=A.Transport(dm.nranks), use_graph=use_graph)
    rn = mg.solve(phi, b, rtol=1e-10, max_iter=100)
    return mg, rn, A.gather_global(phi, dom)


@pytest.mark.parametrize("n,m", [(64, 32), (128, 32), (256, 64), (48, 16), (64, 64), (64, 4), (96, 32)])
def test_hierarchy_resolutions_match_oracle(n, m):
    dom = A.Box((0, 0, 0), (n - 1,) * 3)
    ba = A.BoxArray([dom]).max_size(m)
    dev = [(tuple(d.lo), tuple(d.hi)) for d, b, k in A.mg_hierarchy(dom, ba)]
    ref = [d for d, b, k in R.mg_levels(((0, 0, 0), (n - 1,) * 3), tboxes(ba))]
    assert dev == ref


def test_hierarchy_matches_oracle():
    for n, m in ((64, 32), (128, 32), (256, 64), (48, 16)):
        dom = A.Box((0, 0, 0), (n - 1,) * 3)
        ba = A.BoxArray([dom]).max_size(m)
        dev = [(tuple(d.lo), tuple(d.hi)) for d, b, k in A.mg_hierarchy(dom, ba)]
        ref = [d for d, b, k in R.mg_levels(((0, 0, 0), (n - 1,) * 3), tboxes(ba))]
        # same resolutions; the device agglomerates earlier (one-CTA coarse tail)
        assert dev == ref


@pytest.mark.parametrize("n,m", [(32, 16), (64, 32), (48, 16), (64, 64), (32, 4)])
def test_solve_matches_oracle_bitwise(n, m):
    dom, ba, dm, geom, rhs = _problem(n, m, seed=1)
    ref = R.OracleMLMG(((0, 0, 0), (n - 1,) * 3), tboxes(ba)).solve(rhs, rtol=1e-10, max_iter=100)
    mg, rn, phi = _solve_device(dom, ba, dm, geom, rhs)
    assert mg.iterations == ref["iterations"]
    assert mg.history == ref["history"]
    assert np.array_equal(phi, ref["phi"])


def test_graph_and_eager_agree():
    dom, ba, dm, geom, rhs = _problem(32, 16, seed=5)
    mg1, rn1, phi1 = _solve_device(dom, ba, dm, geom, rhs, use_graph=True)
    mg2, rn2, phi2 = _solve_device(dom, ba, dm, geom, rhs, use_graph=False)
    assert mg1.history == mg2.history and np.array_equal(phi1, phi2)


def test_simulated_ranks_bit_identical():
    dom, ba, dm, geom, rhs = _problem(64, 16, seed=2)
    base = _solve_device(dom, ba, dm, geom, rhs)
    for r in (2, 4, 8):
        mg, rn, phi = _solve_device(dom, ba, dm, geom, rhs, nranks=r)
        assert mg.history == base[0].history and np.array_equal(phi, base[2])


def test_c2_converges_to_1e10():
    """Config C2: 128^3, 32^3 boxes, solve to 1e-10 relative residual."""
    dom, ba, dm, geom, rhs = _problem(128, 32, seed=1)
    mg, rn, phi = _solve_device(dom, ba, dm, geom, rhs)
    assert rn <= 1e-10 * mg.r0
    assert mg.iterations <= 15
    # residual recomputed independently from the returned solution
    p = A.MultiFab(ba, dm, 1, 1)
    p.load_valid_from(dom, phi)
    A.fill_boundary(p, A.Transport(1), dom, True)
    r = A.MultiFab(ba, dm, 1, 0)
    b = A.MultiFab(ba, dm, 1, 0)
    b.load_valid_from(dom, rhs)
    from paper_2009_12009_b200 import stencil as S

    S.residual(r, b, p, S.dh_of(geom))
    assert A.device_reduce(r, "absmax").item() == rn


@pytest.mark.parametrize("n,m", [(64, 32), (64, 64)])
def test_ghost_push_solve_matches_oracle_bitwise(n, m):
    """MLMG(ghost_push=True): prolongation pushes the fine level's ghosts (no
    copy-program fill) -- same iterations, history and solution as the oracle."""
    dom, ba, dm, geom, rhs = _problem(n, m, seed=3)
    ref = R.OracleMLMG(((0, 0, 0), (n - 1,) * 3), tboxes(ba)).solve(rhs, rtol=1e-10, max_iter=100)
    phi = A.MultiFab(ba, dm, 1, 1)
    b = A.MultiFab(ba, dm, 1, 0)
    b.load_valid_from(dom, rhs)
    mg = A.MLMG(geom, ba, dm, transport=A.Transport(1), ghost_push=True)
    assert any(lv.push for lv in mg.levels)
    mg.solve(phi, b, rtol=1e-10, max_iter=100)
    assert mg.iterations == ref["iterations"] and mg.history == ref["history"]
    assert np.array_equal(A.gather_global(phi, dom), ref["phi"])


@pytest.mark.parametrize("n,m", [(64, 32), (128, 128)])
def test_ghost_pull_solve_matches_oracle_bitwise(n, m):
    """MLMG(ghost_pull=True): sweeps whose input ghosts are stale copy them
    themselves (amrb_gsrb_sweep_pull, no copy-program fill before them) --
    same iterations, history and solution as the oracle."""
    dom, ba, dm, geom, rhs = _problem(n, m, seed=4)
    ref = R.OracleMLMG(((0, 0, 0), (n - 1,) * 3), tboxes(ba)).solve(rhs, rtol=1e-10, max_iter=100)
    phi = A.MultiFab(ba, dm, 1, 1)
    b = A.MultiFab(ba, dm, 1, 0)
    b.load_valid_from(dom, rhs)
    mg = A.MLMG(geom, ba, dm, transport=A.Transport(1), ghost_pull=True)
    assert any(lv.pull for lv in mg.levels)
    mg.solve(phi, b, rtol=1e-10, max_iter=100)
    assert mg.iterations == ref["iterations"] and mg.history == ref["history"]
    assert np.array_equal(A.gather_global(phi, dom), ref["phi"])


@pytest.mark.parametrize("n,m", [(128, 64), (256, 64)])
def test_fused_prolong_sweep_solve_identical(n, m):
    """MLMG(fuse_prolong=True) (default: prolongation inside the first
    post-smoothing sweep) == fuse_prolong=False, bit for bit, same history."""
    dom, ba, dm, geom, rhs = _problem(n, m, 5)
    out = []
    for fuse in (True, False):
        phi = A.MultiFab(ba, dm, 1, 1)
        b = A.MultiFab(ba, dm, 1, 0)
        b.load_valid_from(dom, rhs)
        mg = A.MLMG(geom, ba, dm, transport=A.Transport(1), fuse_prolong=fuse)
        if fuse:
            assert any(lv.fuse for lv in mg.levels)
        mg.solve(phi, b, rtol=1e-10, max_iter=100)
        if fuse:
            assert any(lv.fuse for lv in mg.levels)  # the fused path ran (no ENOTSUP fallback)
        out.append((mg.iterations, list(mg.history), A.gather_global(phi, dom)))
    assert out[0][0] == out[1][0]
    assert out[0][1] == out[1][1]
    assert np.array_equal(out[0][2], out[1][2])


@pytest.mark.parametrize("n,m", [(64, 32), (128, 64), (256, 64)])
def test_cluster_tail_solve_identical(n, m):
    """MLMG(cluster_tail=True) (default: the 32^3 level joins the coarse tail on
    an 8-CTA cluster) == cluster_tail=False, bit for bit, same history; at 64^3
    also == the oracle."""
    dom, ba, dm, geom, rhs = _problem(n, m, 7)
    out = []
    for ct in (True, False):
        phi = A.MultiFab(ba, dm, 1, 1)
        b = A.MultiFab(ba, dm, 1, 0)
        b.load_valid_from(dom, rhs)
        mg = A.MLMG(geom, ba, dm, transport=A.Transport(1), cluster_tail=ct)
        assert mg.cluster_tail == ct
        mg.solve(phi, b, rtol=1e-10, max_iter=100)
        out.append((mg.iterations, list(mg.history), A.gather_global(phi, dom)))
    assert out[0][0] == out[1][0]
    assert out[0][1] == out[1][1]
    assert np.array_equal(out[0][2], out[1][2])
    if n == 64:
        ref = R.OracleMLMG(((0, 0, 0), (n - 1,) * 3), tboxes(ba)).solve(rhs, rtol=1e-10, max_iter=100)
        assert out[0][0] == ref["iterations"] and out[0][1] == ref["history"]
        assert np.array_equal(out[0][2], ref["phi"])


_REF = {}


@pytest.mark.parametrize("ct,gcells", [(True, 64**3), (False, 64**3), (True, 0), (False, 128**3)])
def test_grid_levels_solve_matches_oracle(ct, gcells):
    """Small single-box levels as one grid-synchronised launch per half cycle
    (amrb_level_grid), alone, chained (64^3 -> 32^3 above the one-CTA tail) and
    off, with and without the cluster tail: same iterations, history and
    bit-identical solution as the oracle (128^3, 64^3 boxes)."""
    n, m = 128, 64
    dom, ba, dm, geom, rhs = _problem(n, m, 11)
    if "r128" not in _REF:  # one oracle solve (~11 s) shared by the cases
        _REF["r128"] = R.OracleMLMG(((0, 0, 0), (n - 1,) * 3), tboxes(ba)).solve(rhs, rtol=1e-10, max_iter=100)
    ref = _REF["r128"]
    phi = A.MultiFab(ba, dm, 1, 1)
    b = A.MultiFab(ba, dm, 1, 0)
    b.load_valid_from(dom, rhs)
    mg = A.MLMG(geom, ba, dm, transport=A.Transport(1), cluster_tail=ct, grid_level_cells=gcells)
    ngrid = mg.tail - mg.grid_from
    assert ngrid == (0 if gcells == 0 else (1 if ct else 2))
    mg.solve(phi, b, rtol=1e-10, max_iter=100)
    assert mg.iterations == ref["iterations"] and mg.history == ref["history"]
    assert np.array_equal(A.gather_global(phi, dom), ref["phi"])


def test_grid_and_cluster_levels_eager_equals_graph():
    """The cooperative grid-level and cluster-tail launches behave the same
    eagerly (PDL on the neighbouring launches) and inside the captured graph."""
    dom, ba, dm, geom, rhs = _problem(128, 64, seed=13)
    mg1, rn1, phi1 = _solve_device(dom, ba, dm, geom, rhs, use_graph=True)
    mg2, rn2, phi2 = _solve_device(dom, ba, dm, geom, rhs, use_graph=False)
    assert mg1.cluster_tail and mg1.tail > mg1.grid_from
    assert mg1.history == mg2.history and np.array_equal(phi1, phi2)


@pytest.mark.parametrize("mode", [1, 2, 0])
@pytest.mark.parametrize("shape", [(64, 32, 32), (32, 64, 32), (64, 64, 32)])
def test_noncubic_pow2_tail_matches_oracle(shape, mode):
    """Non-cubic power-of-two coarse chains (the multi-GPU weak-scaling shapes)
    take k_coarse_tail_p2x (or, with cluster_tail=2, k_coarse_tail_cl for a
    32 x n1 x n2 top level; 0: no cluster kernel) and grid levels above: same
    iterations, history and bit-identical solution as the oracle."""
    hi = tuple(s - 1 for s in shape)
    dom = A.Box((0, 0, 0), hi)
    ba = A.BoxArray([dom]).max_size(32)
    dm = A.DistributionMapping.single_rank(len(ba))
    geom = A.Geometry(dom, (0.0,) * 3, tuple(s / 32.0 for s in shape), True)
    rng = np.random.default_rng(17)
    rhs = rng.standard_normal(shape)
    rhs -= rhs.mean()
    ref = R.OracleMLMG(((0, 0, 0), hi), tboxes(ba), prob_hi=tuple(s / 32.0 for s in shape)).solve(
        rhs, rtol=1e-10, max_iter=100)
    phi = A.MultiFab(ba, dm, 1, 1)
    b = A.MultiFab(ba, dm, 1, 0)
    b.load_valid_from(dom, rhs)
    mg = A.MLMG(geom, ba, dm, transport=A.Transport(1), cluster_tail=mode)
    assert mg.tail < len(mg.levels)
    # the non-cubic cluster tail needs cluster_tail=2 (the default); 1 = cubic only
    assert mg.cluster_tail == (mode == 2 and shape[0] == 64)
    mg.solve(phi, b, rtol=1e-10, max_iter=100)
    assert mg.iterations == ref["iterations"] and mg.history == ref["history"]
    assert np.array_equal(A.gather_global(phi, dom), ref["phi"])


@pytest.mark.parametrize("per,value,n,m", [((False, False, False), 0.0, 64, 32), ((True, False, False), 1.5, 64, 32),
                                          ((False, True, False), -0.25, 48, 16), ((False, False, False), 0.5, 64, 64)])
def test_external_boundary_solve_matches_oracle(per, value, n, m):
    """Non-periodic MLMG: 'external' sides (BoundaryRecord, amr_core.py:73-108)
    hold `value` in the finest level's ghosts; the coarse correction levels use
    the level-consistent homogeneous ghosts of oracle/mlmg_ref.py
    (reflect_ghosts).  Same iterations, history and bit-identical solution."""
    dom = A.Box((0, 0, 0), (n - 1,) * 3)
    ba = A.BoxArray([dom]).max_size(m)
    dm = A.DistributionMapping.single_rank(len(ba))
    geom = A.Geometry(dom, (0.0,) * 3, (1.0,) * 3, per)
    conds = tuple("periodic" if p else "external" for p in per)
    bc = A.BoundaryRecord(conds, conds, value)
    rng = np.random.default_rng(23)
    rhs = rng.standard_normal((n, n, n))
    ref = R.OracleMLMG(((0, 0, 0), (n - 1,) * 3), tboxes(ba), bc=(conds, conds, value)).solve(
        rhs, rtol=1e-10, max_iter=60)
    phi = A.MultiFab(ba, dm, 1, 1)
    b = A.MultiFab(ba, dm, 1, 0)
    b.load_valid_from(dom, rhs)
    mg = A.MLMG(geom, ba, dm, transport=A.Transport(1), bc=bc)
    assert mg.tail == len(mg.levels) and not any(lv.fuse for lv in mg.levels)
    mg.solve(phi, b, rtol=1e-10, max_iter=60)
    assert mg.iterations == ref["iterations"] and mg.history == ref["history"]
    assert np.array_equal(A.gather_global(phi, dom), ref["phi"])


def test_mlmg_boundary_arguments():
    dom = A.Box((0, 0, 0), (31, 31, 31))
    ba = A.BoxArray([dom])
    dm = A.DistributionMapping.single_rank(1)
    with pytest.raises(ValueError):  # non-periodic geometry without a record
        A.MLMG(A.Geometry(dom, (0.0,) * 3, (1.0,) * 3, False), ba, dm)
    with pytest.raises(ValueError):  # extrap sides are not supported by the solver
        A.MLMG(A.Geometry(dom, (0.0,) * 3, (1.0,) * 3, False), ba, dm, bc=A.BoundaryRecord.all_extrap(3))
    with pytest.raises(ValueError):  # record disagrees with the geometry's periodic flags
        A.MLMG(A.Geometry(dom, (0.0,) * 3, (1.0,) * 3, True), ba, dm,
               bc=A.BoundaryRecord(("external",) * 3, ("external",) * 3))


def test_max_iter_and_repeated_solves_follow_the_oracle():
    """The WHILE-graph loop's state (device memory, reset by a kernel before
    each launch): max_iter stops it exactly where the oracle stops, a second
    solve of the same problem replays the same bits, max_iter=0 only returns
    ||rhs|| and out-of-range max_iter is rejected."""
    n, m = 64, 32
    dom, ba, dm, geom, rhs = _problem(n, m, seed=21)
    ref3 = R.OracleMLMG(((0, 0, 0), (n - 1,) * 3), tboxes(ba)).solve(rhs, rtol=1e-10, max_iter=3)
    b = A.MultiFab(ba, dm, 1, 0)
    b.load_valid_from(dom, rhs)
    mg = A.MLMG(geom, ba, dm, transport=A.Transport(1))
    out = []
    for _ in range(2):
        phi = A.MultiFab(ba, dm, 1, 1)
        rn = mg.solve(phi, b, rtol=1e-10, max_iter=3)
        out.append((mg.iterations, list(mg.history), rn, A.gather_global(phi, dom)))
    assert mg.graph_replays == 2
    for it, hist, rn, phi in out:
        assert it == 3 == ref3["iterations"] and hist == ref3["history"] and rn == hist[-1]
        assert np.array_equal(phi, ref3["phi"])
    phi = A.MultiFab(ba, dm, 1, 1)
    r0 = mg.solve(phi, b, rtol=1e-10, max_iter=0)
    assert mg.iterations == 0 and mg.history == [] and r0 == float(np.abs(rhs).max())
    with pytest.raises(ValueError):
        mg.solve(phi, b, max_iter=mg._HIST + 1)


@pytest.mark.parametrize("shape", [(128, 64, 32), (64, 128, 64), (32, 32, 128)])
def test_noncubic_single_box_solve_matches_oracle(shape):
    """A non-cubic domain in ONE box (the solver's levels are one periodic box
    each: the record-free wrap fill, streaming sweeps, grid levels and tail):
    same iterations, history and bit-identical solution as the oracle."""
    hi = tuple(s - 1 for s in shape)
    dom = A.Box((0, 0, 0), hi)
    ba = A.BoxArray([dom])
    dm = A.DistributionMapping.single_rank(1)
    prob_hi = tuple(s / 64.0 for s in shape)
    geom = A.Geometry(dom, (0.0,) * 3, prob_hi, True)
    rng = np.random.default_rng(23)
    rhs = rng.standard_normal(shape)
    rhs -= rhs.mean()
    ref = R.OracleMLMG(((0, 0, 0), hi), tboxes(ba), prob_hi=prob_hi).solve(rhs, rtol=1e-10, max_iter=100)
    phi = A.MultiFab(ba, dm, 1, 1)
    b = A.MultiFab(ba, dm, 1, 0)
    b.load_valid_from(dom, rhs)
    mg = A.MLMG(geom, ba, dm, transport=A.Transport(1))
    mg.solve(phi, b, rtol=1e-10, max_iter=100)
    assert mg.iterations == ref["iterations"] and mg.history == ref["history"]
    assert np.array_equal(A.gather_global(phi, dom), ref["phi"])


def test_queued_solves_equal_synchronous_solves():
    """solve(wait=False) queues a solve on the stream; finish() returns the
    oldest one's ||r|| and sets its iterations / history.  Two queued solves
    of different right-hand sides give the synchronous solves' bits."""
    n, m = 64, 32
    dom, ba, dm, geom, rhs1 = _problem(n, m, seed=31)
    rhs2 = np.random.default_rng(32).standard_normal((n, n, n))
    rhs2 -= rhs2.mean()
    mg = A.MLMG(geom, ba, dm, transport=A.Transport(1))
    sync = []
    for r in (rhs1, rhs2):
        b = A.MultiFab(ba, dm, 1, 0)
        b.load_valid_from(dom, r)
        phi = A.MultiFab(ba, dm, 1, 1)
        rn = mg.solve(phi, b, rtol=1e-10, max_iter=100)
        sync.append((rn, mg.iterations, list(mg.history), A.gather_global(phi, dom)))
    bs, phis = [], []
    for r in (rhs1, rhs2):
        b = A.MultiFab(ba, dm, 1, 0)
        b.load_valid_from(dom, r)
        bs.append(b)
        phis.append(A.MultiFab(ba, dm, 1, 1))
    assert mg.solve(phis[0], bs[0], rtol=1e-10, max_iter=100, wait=False) is None
    assert mg.solve(phis[1], bs[1], rtol=1e-10, max_iter=100, wait=False) is None
    with pytest.raises(RuntimeError):
        mg.solve(phis[1], bs[1], wait=False)  # at most two queued
    for (rn, it, hist, phi_ref), phi in zip(sync, phis):
        assert mg.finish() == rn and mg.iterations == it and mg.history == hist
        assert np.array_equal(A.gather_global(phi, dom), phi_ref)
    with pytest.raises(RuntimeError):
        mg.finish()
