"""MLMG parity at the headline configs (BASELINE.json configs[1], configs[2]).

C2 (128^3, 32^3 boxes, seed 1) and C3 (256^3, 64^3 boxes, seed 2 -- the
config bench.py's metric is quoted on) are solved through the public
``MLMG.solve`` and compared with the CPU oracle's solve of the SAME rhs bits
(tests/golden/mlmg_golden.json, written by tests/golden/make_mlmg_golden.py
from oracle.mlmg_ref.OracleMLMG): iteration count, the residual history (every
value bit for bit), r0, and the converged solution (sha256 of the gathered
global array plus a probe lattice that localises a mismatch).

The Dirichlet variant (every side BoundaryRecord 'external', value 0,
amr_core.py:73-146) of C2 is pinned the same way.
"""

import hashlib
import json
import os

import numpy as np
import pytest

import paper_2009_12009_b200 as A
from golden.make_mlmg_golden import headline_rhs

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = json.load(open(os.path.join(HERE, "golden", "mlmg_golden.json")))


def _sha(a):
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.float64).tobytes()).hexdigest()


def _rhs(case):
    g = GOLD[case]
    rhs = headline_rhs(g["n"], g["seed"], centre=g["bc"] == "periodic")
    assert _sha(rhs) == g["rhs_sha256"], "numpy generated different rhs bits than the golden run"
    return rhs


@pytest.mark.parametrize("case", sorted(GOLD))
def test_golden_rhs_reproducible(case):
    """CPU: the generator recipe reproduces the golden rhs bits on this host."""
    _rhs(case)


@pytest.mark.gpu
@pytest.mark.parametrize("case", sorted(GOLD))
def test_headline_solve_matches_oracle(case):
    g = GOLD[case]
    n, m = g["n"], g["box"]
    rhs = _rhs(case)
    dom = A.Box((0, 0, 0), (n - 1,) * 3)
    ba = A.BoxArray([dom]).max_size(m)
    dm = A.DistributionMapping.single_rank(len(ba))
    periodic = g["bc"] == "periodic"
    geom = A.Geometry(dom, (0.0,) * 3, (1.0,) * 3, periodic)
    bc = None if periodic else A.BoundaryRecord(("external",) * 3, ("external",) * 3, 0.0)
    b = A.MultiFab(ba, dm, 1, 0)
    b.load_valid_from(dom, rhs)
    phi = A.MultiFab(ba, dm, 1, 1)
    mg = A.MLMG(geom, ba, dm, transport=A.Transport(1), bc=bc)
    rn = mg.solve(phi, b, rtol=g["rtol"], max_iter=200)
    assert float(mg.r0).hex() == g["r0"]
    assert mg.iterations == g["iterations"]
    assert [float(x).hex() for x in mg.history] == g["history"]
    assert float(rn).hex() == g["history"][-1]
    out = A.gather_global(phi, dom)
    s = g["phi_probe_stride"]
    assert [float(x).hex() for x in out[::s, ::s, ::s].ravel()] == g["phi_probe"]
    assert _sha(out) == g["phi_sha256"]


@pytest.mark.gpu
@pytest.mark.parametrize("nranks", [2, 8])
def test_c2_on_simulated_ranks_matches_oracle(nranks):
    """C2 with the boxes spread over 2 / 8 simulated ranks (Morton SFC, the C4
    decomposition): the solver re-boxes one octant per rank and still returns
    the oracle's iterations, history and solution bit for bit."""
    g = GOLD["c2"]
    n, m = g["n"], g["box"]
    rhs = _rhs("c2")
    dom = A.Box((0, 0, 0), (n - 1,) * 3)
    ba = A.BoxArray([dom]).max_size(m)
    dm = A.sfc_distribute(ba, A.default_costs(ba), nranks)
    geom = A.Geometry(dom, (0.0,) * 3, (1.0,) * 3, True)
    b = A.MultiFab(ba, dm, 1, 0)
    b.load_valid_from(dom, rhs)
    phi = A.MultiFab(ba, dm, 1, 1)
    mg = A.MLMG(geom, ba, dm, transport=A.Transport(nranks))
    assert len(mg.levels[0].ba) == nranks  # one box per rank on the solver's levels
    mg.solve(phi, b, rtol=g["rtol"], max_iter=200)
    assert mg.iterations == g["iterations"]
    assert [float(x).hex() for x in mg.history] == g["history"]
    assert _sha(A.gather_global(phi, dom)) == g["phi_sha256"]
