"""Known-answer tests pinning the (reference-unpinned) MLMG definitions of the
oracle: the discrete Laplacian's periodic eigenmodes, a dense 8^3 solve, and
the V-cycle convergence factor (CPU)."""

import numpy as np
import pytest

from oracle import mesh_ref as M
from oracle import mlmg_ref as R


def _ghosted_periodic(u):
    return np.pad(u, 1, mode="wrap")


def test_laplacian_periodic_eigenmode():
    n = 16
    dx = 1.0 / n
    dh = (1.0 / dx**2,) * 3
    x = (np.arange(n) + 0.5) * dx
    for kv in ((1, 0, 0), (1, 2, 0), (3, 1, 2)):
        u = (np.sin(2 * np.pi * kv[0] * x)[:, None, None] * np.cos(2 * np.pi * kv[1] * x)[None, :, None]
             * np.cos(2 * np.pi * kv[2] * x)[None, None, :])
        lam = sum((2 * np.cos(2 * np.pi * k * dx) - 2) / dx**2 for k in kv)
        lu = R.laplacian(_ghosted_periodic(u), dh)
        assert np.allclose(lu, lam * u, rtol=0, atol=1e-9 * abs(lam))


def _dense_operator(n, dh):
    N = n**3
    A = np.zeros((N, N))
    idx = lambda i, j, k: ((i % n) * n + (j % n)) * n + (k % n)  # noqa: E731
    for i in range(n):
        for j in range(n):
            for k in range(n):
                r = idx(i, j, k)
                A[r, r] = -2 * (dh[0] + dh[1] + dh[2])
                for d, (a, b, c) in enumerate(((1, 0, 0), (0, 1, 0), (0, 0, 1))):
                    A[r, idx(i + a, j + b, k + c)] += dh[d]
                    A[r, idx(i - a, j - b, k - c)] += dh[d]
    return A


def test_dense_8cubed_solve_matches_vcycle():
    """8^3 periodic Poisson: the V-cycle solution equals the dense least-squares
    solution (both mean-free) to ~1e-10 of its size."""
    n = 8
    rng = np.random.default_rng(3)
    rhs = rng.standard_normal((n, n, n))
    rhs -= rhs.mean()
    dom = ((0, 0, 0), (n - 1,) * 3)
    boxes = [((i, j, k), (i + 3, j + 3, k + 3)) for i in (0, 4) for j in (0, 4) for k in (0, 4)]
    out = R.OracleMLMG(dom, boxes).solve(rhs, rtol=1e-12, max_iter=100)
    dh = R.level_dh(dom, (0.0,) * 3, (1.0,) * 3)
    A = _dense_operator(n, dh)
    ref = np.linalg.lstsq(A, rhs.ravel(), rcond=None)[0].reshape(n, n, n)
    phi = out["phi"] - out["phi"].mean()
    ref = ref - ref.mean()
    assert np.abs(phi - ref).max() <= 1e-9 * np.abs(ref).max()


@pytest.mark.parametrize("n,m", [(32, 16), (64, 32)])
def test_vcycle_convergence_factor(n, m):
    rng = np.random.default_rng(1)
    rhs = rng.standard_normal((n, n, n))
    rhs -= rhs.mean()
    boxes = [((i, j, k), (i + m - 1, j + m - 1, k + m - 1)) for i in range(0, n, m) for j in range(0, n, m)
             for k in range(0, n, m)]
    out = R.OracleMLMG(((0, 0, 0), (n - 1,) * 3), boxes).solve(rhs, rtol=1e-10, max_iter=40)
    h = np.array([out["r0"]] + out["history"])
    rates = h[1:] / h[:-1]
    assert out["history"][-1] <= 1e-10 * out["r0"]
    assert rates[1:].max() < 0.2
    assert out["iterations"] <= 12


def test_gsrb_one_colour_touches_only_that_colour():
    n = 6
    rng = np.random.default_rng(2)
    p = rng.standard_normal((n + 2,) * 3)
    before = p.copy()
    R.gsrb_color(((0, 0, 0), (n - 1,) * 3), p, rng.standard_normal((n,) * 3), (1.0, 1.0, 1.0), 0)
    changed = p[1:-1, 1:-1, 1:-1] != before[1:-1, 1:-1, 1:-1]
    i, j, k = np.indices((n,) * 3)
    assert not changed[(i + j + k) % 2 == 1].any()
    assert changed[(i + j + k) % 2 == 0].all()


def test_hierarchy_levels():
    dom = ((0, 0, 0), (255, 255, 255))
    boxes = [((i, j, k), (i + 63, j + 63, k + 63)) for i in range(0, 256, 64) for j in range(0, 256, 64)
             for k in range(0, 256, 64)]
    lv = R.mg_levels(dom, boxes)
    assert [M.ext(d)[0] for d, _, _ in lv] == [256, 128, 64, 32, 16, 8, 4]
    assert [k for _, _, k in lv] == ["base", "boxlocal", "boxlocal", "boxlocal", "boxlocal", "agglom", "single"]


def test_threaded_oracle_is_bit_identical():
    """The thread-pooled per-box loops (bench.py's reference arm) give the same
    bits, iteration count and residual history as the serial oracle."""
    n, m = 32, 8
    rng = np.random.default_rng(5)
    rhs = rng.standard_normal((n, n, n))
    rhs -= rhs.mean()
    boxes = [((i, j, k), (i + m - 1, j + m - 1, k + m - 1)) for i in range(0, n, m) for j in range(0, n, m)
             for k in range(0, n, m)]
    dom = ((0, 0, 0), (n - 1,) * 3)
    a = R.OracleMLMG(dom, boxes).solve(rhs, rtol=1e-10, max_iter=40)
    b = R.OracleMLMG(dom, boxes, threads=4).solve(rhs, rtol=1e-10, max_iter=40)
    assert a["iterations"] == b["iterations"]
    assert a["history"] == b["history"]
    assert np.array_equal(a["phi"], b["phi"])


@pytest.mark.parametrize("ext,m,nranks", [((256, 256, 256), 64, 1), ((128, 128, 128), 32, 1), ((512, 256, 256), 64, 2),
                                          ((512, 512, 256), 64, 4), ((512, 512, 512), 64, 8), ((96, 64, 128), 32, 1),
                                          ((64, 32, 32), 32, 1), ((48, 48, 48), 16, 1)])
def test_device_hierarchy_has_the_oracle_resolutions(ext, m, nranks):
    """mlmg.mg_hierarchy (the device solver's levels: it agglomerates earlier,
    into replicated or one-box levels) keeps the oracle's level RESOLUTIONS
    (oracle/mlmg_ref.py mg_levels) -- the box decomposition of a level does not
    change its values, so the V-cycles stay bit-identical."""
    import paper_2009_12009_b200 as A
    from paper_2009_12009_b200.mlmg import mg_hierarchy

    dom = A.Box((0, 0, 0), tuple(e - 1 for e in ext))
    ba = A.BoxArray([dom]).max_size(m)
    dev = [tuple(d.extents()) for d, _, _ in mg_hierarchy(dom, ba, nranks)]
    boxes = [(tuple(b.lo), tuple(b.hi)) for b in ba]
    ref = [tuple(M.ext(d)) for d, _, _ in R.mg_levels(((0, 0, 0), tuple(e - 1 for e in ext)), boxes)]
    assert dev == ref
