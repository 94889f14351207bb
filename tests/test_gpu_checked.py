"""Checked build (make -C paper_2009_12009_b200/csrc CHECKED=1): every
concurrency-heavy kernel path of tools/sanitize.py -- the streaming sweep in
all modes with and without ghost push (TMA ring, mbarriers, proxy fences, one
barrier per step, both stream directions), the cluster coarse tail (DSMEM),
the grid-synchronised level, copy-program fills and the WHILE-graph solve --
runs with its device-side invariant checks on and records no failure.
compute-sanitizer is closed on this GPU pool (profiles/r2_sanitizer.txt).

Also: repeated launches of the streaming sweep are bit-identical (a data race
between its warps would show up as run-to-run differences)."""

import os
import subprocess
import sys

import numpy as np
import pytest
import torch

import paper_2009_12009_b200 as A
from paper_2009_12009_b200 import stencil as S

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_checked_build_records_no_failures():
    lib = os.path.join(ROOT, "paper_2009_12009_b200", "_lib", "libamrb_checked.so")
    assert os.path.exists(lib), "checked build missing (make -C paper_2009_12009_b200/csrc CHECKED=1)"
    env = dict(os.environ, AMRB_LIBRARY="checked")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "sanitize.py")], env=env, capture_output=True,
                         text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    assert "libamrb_checked.so: DCHECK failures 0" in out.stdout, out.stdout[-2000:]


@pytest.mark.parametrize("n,m", [(128, 128), (64, 32)])
def test_stream_sweep_repeatable(n, m):
    dom = A.Box((0, 0, 0), (n - 1,) * 3)
    ba = A.BoxArray([dom]).max_size(m)
    dm = A.DistributionMapping.single_rank(len(ba))
    tr = A.Transport(1)
    a, rhs = A.MultiFab(ba, dm, 1, 2), A.MultiFab(ba, dm, 1, 1)
    rng = np.random.default_rng(3)
    a.load_valid_from(dom, rng.normal(size=(n, n, n)))
    rhs.load_valid_from(dom, rng.normal(size=(n, n, n)))
    A.fill_boundary(a, tr, dom, True)
    A.fill_boundary(rhs, tr, dom, True)
    outs = []
    for _ in range(12):
        b = A.MultiFab(ba, dm, 1, 2)
        S.gsrb_sweep(a, b, rhs, (4096.0,) * 3)
        outs.append(b.storage.clone())
    torch.cuda.synchronize()
    assert all(torch.equal(outs[0], o) for o in outs[1:])
