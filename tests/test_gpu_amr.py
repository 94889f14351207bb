"""Two-level subcycled advection on device: fill_patch (time
blend + limited-linear interpolation + fine-wins copy), FluxRegister
(crse_add / fine_add / reflux) and the upwind update, checked bit for bit
against the reference's own AdvectionSolver (fixtures from
tests/golden/make_golden.py) and for conservation to 1e-12."""

import os

import numpy as np
import pytest

import paper_2009_12009_b200 as A
from paper_2009_12009_b200 import amr

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _setup(name, reflux):
    g = np.load(os.path.join(GOLD, f"{name}.npz"))
    dim, n, nranks = (int(x) for x in g["meta"])
    dom = A.Box(A.IntVect([0] * dim), A.IntVect([n - 1] * dim))
    geom = A.Geometry(dom, (0.0,) * dim, (1.0,) * dim, (True,) * dim)
    bas, dms = [], []
    for lev in (0, 1):
        boxes = [A.Box(A.IntVect(r[:dim]), A.IntVect(r[dim:])) for r in g[f"ba{lev}"].tolist()]
        bas.append(A.BoxArray(boxes))
        dms.append(A.DistributionMapping(list(g[f"dm{lev}"]), nranks))
    s = amr.AdvectionSolver(geom, bas[0], dms[0], bas[1], dms[1], tuple(g["ratio"]), tuple(g["velocity"]),
                            cfl=float(g["cfl"]), use_reflux=reflux)
    for lev in (0, 1):
        for i in range(len(bas[lev])):
            s.phi[lev].fab(i).valid().copy_(
                __import__("torch").as_tensor(g[f"r_s0_L{lev}_b{i}"]))
    return g, s


@pytest.mark.parametrize("name", ["adv2d", "adv3d"])
@pytest.mark.parametrize("reflux", [True, False])
def test_advection_matches_reference_bitwise(name, reflux):
    g, s = _setup(name, reflux)
    tag = "r" if reflux else "n"
    done = 0
    for st in [int(x) for x in g["steps"]][1:]:
        while done < st:
            s.step()
            done += 1
        assert s.time == float(g[f"{tag}_s{st}_time"])
        for lev in (0, 1):
            for i in range(len(s.phi[lev].ba)):
                got = s.phi[lev].fab(i).valid().cpu().numpy()
                want = g[f"{tag}_s{st}_L{lev}_b{i}"]
                assert np.array_equal(got, want), (name, reflux, st, lev, i, np.abs(got - want).max())
        assert s.total_mass() == pytest.approx(float(g[f"{tag}_s{st}_mass"]), rel=1e-14, abs=0)


def test_conservation_criterion_06():
    """test_acceptance.py:403-428: 100 subcycled steps conserve to 1e-12 with
    refluxing, and do not without it."""
    for reflux, ok in ((True, True), (False, False)):
        g, s = _setup("adv2d", reflux)
        m0 = s.total_mass()
        for _ in range(100):
            s.step()
        drift = abs(s.total_mass() - m0) / abs(m0)
        assert (drift <= 1e-12) == ok, (reflux, drift)


def test_replayed_steps_count_transport_traffic():
    """Steps 3+ replay a CUDA graph; the per-step transport_messages /
    transport_bytes tallies (counters.py, transport.py:40-58) still grow by
    the same amounts as an eager step's."""
    from paper_2009_12009_b200 import counters

    g, s = _setup("adv2d", True)
    deltas = []
    for _ in range(5):
        b = counters.snapshot()
        s.step()
        a = counters.snapshot()
        deltas.append(tuple(a.get(k, 0) - b.get(k, 0) for k in ("transport_messages", "transport_bytes")))
    assert s._graph is not None
    # step 0 also checks the hierarchy; steps 1 (eager), 2 (captured) and 3, 4
    # (replayed) move the same traffic
    assert len(set(deltas[1:])) == 1, deltas
