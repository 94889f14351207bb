"""numpy restatement of the MLMG Poisson V-cycle (definitions for the device path).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

PARITY UNPINNED: the reference package has no linear solver (SPEC.md:13,
SPEC.md:532); the Laplacian, GSRB smoother, residual and V-cycle are DEFINED
here on top of the reference-pinned primitives in oracle.mesh_ref
(fill_boundary, average_down, interp_to_fine 'pc', reduce), following
SURVEY.md section 8(c):

* operator  L(phi) = (dh0*((phi[i-1]-2phi)+phi[i+1]) + dh1*(...)) + dh2*(...),
  dh_d = 1/dx_d^2, dx from Geometry.cell_size (amr_core.py:37-40);
* residual  r = rhs - L(phi);
* GSRB      per colour c in (0, 1), cells with (i+j+k+c) % 2 == 0 in GLOBAL
  index space: phi <- phi + (rhs - L(phi)) * rgamma with rgamma = 1/gamma,
  gamma = -2*(dh0+dh1+dh2) (the reciprocal is formed once, as upstream AMReX's
  gsrb does with omega/gamma);
  one sweep = fill; colour 0; fill; colour 1 (width-1 fills);
* hierarchy coarsen box-locally by 2 while every box extent is even and >= 8;
  then, if several boxes remain and the domain is still coarsenable (even,
  >= 8), agglomerate onto one box covering the coarsened domain; keep
  coarsening that box while it is even and >= 8.  Restriction = average_down,
  prolongation = phi_f += interp_to_fine(phi_c, 'pc');
* cycle     V(nu1, nu2); coarse-level phi starts at 0; bottom = a fixed number
  of GSRB sweeps; stop when ||r||_inf <= rtol * ||rhs||_inf (phi0 = 0) or
  after max_iter cycles.

Known-answer tests (tests/test_oracle_mlmg.py) pin the discretisation:
discrete periodic eigenmodes, a dense 8^3 solve and the per-cycle
convergence factor.
"""

from __future__ import annotations

from concurrent.futures import ThreadPoolExecutor

import numpy as np

from . import mesh_ref as M

__all__ = ["mg_levels", "level_dh", "laplacian", "gsrb_color", "OracleMLMG", "coarsenable_extent"]


def coarsenable_extent(e):
    return e % 2 == 0 and e >= 8


def mg_levels(domain, boxes):
    """[(domain, boxes, kind)] from fine to coarse; kind in base/boxlocal/agglom/single."""
    two = tuple(2 for _ in domain[0])
    levels = [(domain, list(boxes), "base")]
    while all(coarsenable_extent(e) for b in boxes for e in M.ext(b)):
        boxes = [M.coarsen_box(b, two) for b in boxes]
        domain = M.coarsen_box(domain, two)
        levels.append((domain, boxes, "boxlocal"))
    if len(boxes) > 1 and all(coarsenable_extent(e) for e in M.ext(domain)):
        domain = M.coarsen_box(domain, two)
        boxes = [domain]
        levels.append((domain, boxes, "agglom"))
    while len(boxes) == 1 and all(coarsenable_extent(e) for e in M.ext(domain)):
        domain = M.coarsen_box(domain, two)
        boxes = [domain]
        levels.append((domain, boxes, "single"))
    return levels


def level_dh(domain, prob_lo, prob_hi):
    """1/dx^2 per axis from Geometry.cell_size = (hi - lo)/extent (amr_core.py:37-40)."""
    out = []
    for l, h, e in zip(prob_lo, prob_hi, M.ext(domain)):
        cs = (h - l) / e
        out.append(1.0 / (cs * cs))
    return tuple(out)


def gamma_of(dh):
    return -2.0 * (dh[0] + dh[1] + dh[2])


def rgamma_of(dh):
    return 1.0 / gamma_of(dh)


def laplacian(p, dh):
    """L(phi) over the valid region of a ghost-1 array p of shape (n0+2, n1+2, n2+2)."""
    c = p[1:-1, 1:-1, 1:-1]
    c2 = 2.0 * c
    tx = dh[0] * ((p[:-2, 1:-1, 1:-1] - c2) + p[2:, 1:-1, 1:-1])
    ty = dh[1] * ((p[1:-1, :-2, 1:-1] - c2) + p[1:-1, 2:, 1:-1])
    tz = dh[2] * ((p[1:-1, 1:-1, :-2] - c2) + p[1:-1, 1:-1, 2:])
    return (tx + ty) + tz


_masks = {}


def color_mask(lo, shape, color):
    key = ((lo[0] + lo[1] + lo[2] + color) & 1, shape)
    m = _masks.get(key)
    if m is None:
        i, j, k = np.indices(shape, sparse=True)
        m = ((i + j + k + key[0]) % 2) == 0
        _masks[key] = m
    return m


def gsrb_color(box, p, rhs_valid, dh, color):
    """One colour of GSRB on one box in place (p: ghost-1 array, no comp axis).

    Red cells read only black neighbours, so evaluating L on all cells and
    keeping the coloured ones equals the sequential definition."""
    c = p[1:-1, 1:-1, 1:-1]
    new = c + (rhs_valid - laplacian(p, dh)) * rgamma_of(dh)
    np.copyto(c, new, where=color_mask(box[0], c.shape, color))


def reflect_alpha(level):
    """Coarse-level homogeneous Dirichlet factor: ghost = -alpha * mirror."""
    r = float(1 << level)
    return (r - 1.0) / (r + 1.0)


def reflect_ghosts(boxes, fabs, ngrow, domain, lo_conds, hi_conds, alpha):
    """Every ghost cell outside an 'external' face (ghost layer t = 1..ngrow)
    <- -alpha * the valid cell mirrored across that face (layer t-1 inside),
    one (axis, side) at a time in the order of apply_domain_boundary
    (amr_core.py:118-146); cells outside two faces (edges / corners, never read
    by the 7-point operator) take the last axis' value.  The product is the
    single rounded operation (-alpha) * x."""
    dim = len(domain[0])
    na = -alpha
    for i, b in enumerate(boxes):
        f = fabs[i]
        g = M.grow(b, ngrow)
        for d in range(dim):
            n = g[1][d] - g[0][d] + 1
            for side, cond in (("lo", lo_conds[d]), ("hi", hi_conds[d])):
                if cond == "periodic":
                    continue
                width = domain[0][d] - g[0][d] if side == "lo" else g[1][d] - domain[1][d]
                for t in range(1, width + 1):
                    o = [slice(None)] * (dim + 1)
                    m = [slice(None)] * (dim + 1)
                    if side == "lo":
                        o[1 + d] = slice(width - t, width - t + 1)
                        m[1 + d] = slice(width + t - 1, width + t)
                    else:
                        o[1 + d] = slice(n - width + t - 1, n - width + t)
                        m[1 + d] = slice(n - width - t, n - width - t + 1)
                    f[tuple(o)] = na * f[tuple(m)]


class OracleMLMG:
    """CPU V-cycle solver; data per level as mesh_ref dicts (ncomp = 1)."""

    def __init__(self, domain, boxes, prob_lo=(0.0, 0.0, 0.0), prob_hi=(1.0, 1.0, 1.0), nu1=2, nu2=2,
                 bottom_sweeps=32, threads=1, bc="periodic"):
        """bc: "periodic" (all periodic, the SURVEY 8(c) parity case),
        "dirichlet" (every side BoundaryRecord 'external' with value 0), or
        (lo_conds, hi_conds, value) with per-dimension 'periodic' / 'external'
        conditions (a dimension is periodic iff both its sides are).  After
        every fill the ghost cells outside the domain take the external value
        on the finest level (apply_domain_boundary, amr_core.py:111-146,
        mesh_ref.apply_domain_boundary): the boundary value sits at the ghost
        cell centre, h/2 outside the face.  The coarse levels solve the
        homogeneous correction equation with the boundary at that SAME point:
        level l (spacing H = 2^l h) sets each outside ghost to
        -alpha_l * (its mirror cell across the face), alpha_l = (H-h)/(H+h)
        (linear interpolation through the ghost and first interior centres
        vanishes at -h/2) -- see reflect_ghosts.  A plain ghost = 0 on every
        level puts the coarse boundaries at different points and the V-cycle
        diverges at 128^3.

        threads > 1 runs the per-box loops (GSRB colours, residuals, ghost
        fills grouped by destination box) on a thread pool; numpy releases the
        GIL inside the array ops and boxes of one phase are independent, so the
        results are bit-identical to threads=1 (tests/test_oracle_mlmg.py)."""
        if bc == "periodic":
            bc = (("periodic",) * 3, ("periodic",) * 3, 0.0)
        elif bc == "dirichlet":
            bc = (("external",) * 3, ("external",) * 3, 0.0)
        lo_c, hi_c, value = bc
        for d in range(3):
            if (lo_c[d] == "periodic") != (hi_c[d] == "periodic") or {lo_c[d], hi_c[d]} - {"periodic", "external"}:
                raise ValueError(f"unsupported boundary conditions {bc!r}")
        self.bc = (tuple(lo_c), tuple(hi_c), float(value))
        self.periodic = tuple(c == "periodic" for c in lo_c)
        self.threads = max(1, int(threads))
        self._pool = ThreadPoolExecutor(self.threads) if self.threads > 1 else None
        self.nu1, self.nu2, self.bottom_sweeps = nu1, nu2, bottom_sweeps
        self.levels = []
        for dom, bxs, kind in mg_levels(domain, boxes):
            self.levels.append(
                {
                    "domain": dom,
                    "boxes": bxs,
                    "kind": kind,
                    "dh": level_dh(dom, prob_lo, prob_hi),
                    "phi": M.make_fabs(bxs, 1, 1),
                    "rhs": M.make_fabs(bxs, 1, 0),
                    "fill": M.fill_records(bxs, 1, dom, self.periodic),
                }
            )
        self.sweeps = 0  # GSRB sweeps performed (all levels)
        self.cell_updates = 0

    # -- primitives ------------------------------------------------------------
    def _map(self, fn, items):
        items = list(items)
        if self._pool is None or len(items) < 2:
            return [fn(x) for x in items]
        return list(self._pool.map(fn, items))

    def fill(self, lv):
        self._fill(lv)
        if not all(self.periodic):
            lo_c, hi_c, value = self.bc
            lev = self.levels.index(lv)
            if lev == 0:
                M.apply_domain_boundary(lv["boxes"], lv["phi"], 1, lv["domain"], lo_c, hi_c, value)
            else:
                reflect_ghosts(lv["boxes"], lv["phi"], 1, lv["domain"], lo_c, hi_c, reflect_alpha(lev))

    def _fill(self, lv):
        if self._pool is None:
            M.execute(lv["fill"], lv["boxes"], lv["phi"], 1, lv["boxes"], lv["phi"], 1)
            return
        # a width-1 fill writes ghost cells only and reads valid cells only, so
        # the two-phase staging of M.execute is not needed; records are applied
        # per destination box in plan order.
        by_dst = lv.get("fill_by_dst")
        if by_dst is None:
            by_dst = {}
            for rec in lv["fill"]:
                by_dst.setdefault(rec[1], []).append(rec)
            lv["fill_by_dst"] = by_dst = list(by_dst.items())
        bx, ph = lv["boxes"], lv["phi"]

        def one(item):
            j, recs = item
            for i, _, ov, s in recs:
                ph[j][(slice(None),) + M.region_index(bx[j], 1, M.shift(ov, s))] = \
                    ph[i][(slice(None),) + M.region_index(bx[i], 1, ov)]

        self._map(one, by_dst)

    def smooth(self, lv, n):
        for _ in range(n):
            for color in (0, 1):
                self.fill(lv)
                self._map(lambda ib: gsrb_color(ib[1], lv["phi"][ib[0]][0], lv["rhs"][ib[0]][0], lv["dh"], color),
                          enumerate(lv["boxes"]))
            self.sweeps += 1
            self.cell_updates += sum(int(np.prod(M.ext(b))) for b in lv["boxes"])

    def residual(self, lv):
        self.fill(lv)
        rs = self._map(lambda i: (lv["rhs"][i][0] - laplacian(lv["phi"][i][0], lv["dh"]))[None],
                       range(len(lv["boxes"])))
        return dict(enumerate(rs))

    def norm_inf(self, fabs, boxes):
        mx = M.reduce(boxes, fabs, 0, "max", 0)
        mn = M.reduce(boxes, fabs, 0, "min", 0)
        return max(mx, -mn)

    # -- cycle -------------------------------------------------------------------
    def vcycle(self):
        L = self.levels
        two = (2, 2, 2)
        for l in range(len(L) - 1):
            lv, nx = L[l], L[l + 1]
            if l > 0:
                for f in lv["phi"].values():
                    f[...] = 0.0
            self.smooth(lv, self.nu1)
            r = self.residual(lv)
            M.average_down(lv["boxes"], r, 0, nx["boxes"], nx["rhs"], 0, two)
        bot = L[-1]
        for f in bot["phi"].values():
            f[...] = 0.0
        self.smooth(bot, self.bottom_sweeps)
        for l in range(len(L) - 2, -1, -1):
            lv, nx = L[l], L[l + 1]
            M.interp_pc(lv["boxes"], lv["phi"], 1, nx["boxes"], nx["phi"], 1, two, add=True)
            self.smooth(lv, self.nu2)

    def solve(self, rhs_global, phi_global=None, rtol=1e-10, max_iter=200, max_cycles=None):
        """Returns dict(phi, iterations, history, r0).  max_cycles bounds the work
        (CPU-baseline samples) without the convergence test."""
        top = self.levels[0]
        dom = top["domain"]
        M.load_global(top["boxes"], top["rhs"], 0, dom, np.asarray(rhs_global)[None])
        if phi_global is None:
            for f in top["phi"].values():
                f[...] = 0.0
        else:
            M.load_global(top["boxes"], top["phi"], 1, dom, np.asarray(phi_global)[None])
        r0 = self.norm_inf(top["rhs"], top["boxes"])
        hist = []
        it = 0
        limit = max_iter if max_cycles is None else max_cycles
        while it < limit:
            self.vcycle()
            it += 1
            rn = self.norm_inf(self.residual(top), top["boxes"])
            hist.append(rn)
            if max_cycles is None and rn <= rtol * r0:
                break
        phi = M.gather(top["boxes"], top["phi"], 1, dom)
        return {"phi": phi, "iterations": it, "history": hist, "r0": r0}
