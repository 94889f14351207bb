"""numpy restatement of the reference's mesh-communication path.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Self-contained: no import
of amrkit and no import of the product package, so it can run on the GPU box
(where /root/reference does not exist) and checks the device path
independently.

Data model (same as the reference's Fab, fabarray.py:28-38): a "level" is a
list of boxes ``(lo, hi)`` (tuples, inclusive) and a dict ``fabs`` mapping box
index -> numpy array of shape (ncomp, *(hi - lo + 1 + 2*ngrow)) in C order.

Each function cites the reference code it restates.
"""

from __future__ import annotations

import itertools

import numpy as np

# ---------------------------------------------------------------------------
# box helpers (index_space.py:172-345)
# ---------------------------------------------------------------------------


def ext(b):
    return tuple(h - l + 1 for l, h in zip(*b))


def meet(a, b):
    lo = tuple(max(x, y) for x, y in zip(a[0], b[0]))
    hi = tuple(min(x, y) for x, y in zip(a[1], b[1]))
    return None if any(h < l for l, h in zip(lo, hi)) else (lo, hi)


def grow(b, g):
    return (tuple(x - g for x in b[0]), tuple(x + g for x in b[1]))


def shift(b, s):
    return (tuple(x + d for x, d in zip(b[0], s)), tuple(x + d for x, d in zip(b[1], s)))


def box_diff(a, core):
    """Slabs of a minus core, dimension 0 first, low side then high side
    (index_space.py:320-345)."""
    m = meet(a, core)
    if m is None:
        return [a]
    lo, hi = list(a[0]), list(a[1])
    out = []
    for d in range(len(lo)):
        if lo[d] < m[0][d]:
            top = hi.copy()
            top[d] = m[0][d] - 1
            out.append((tuple(lo), tuple(top)))
            lo[d] = m[0][d]
        if hi[d] > m[1][d]:
            bot = lo.copy()
            bot[d] = m[1][d] + 1
            out.append((tuple(bot), tuple(hi)))
            hi[d] = m[1][d]
    return out


def periodic_shifts(domain, periodic):
    """fabarray.py:235-243 (order irrelevant after the record sort)."""
    e = ext(domain)
    choices = [(-e[d], 0, e[d]) if periodic[d] else (0,) for d in range(len(e))]
    return [tuple(s) for s in itertools.product(*choices)]


# ---------------------------------------------------------------------------
# plans (fabarray.py:169-318, coarse_fine.py:201-220)
# ---------------------------------------------------------------------------


def _sort(records):
    # CommPlan order: (dst index, dst lo, src index, shift)  fabarray.py:182-197
    return sorted(records, key=lambda r: (r[1], tuple(a + s for a, s in zip(r[2][0], r[3])), r[0], r[3]))


def _overlaps(boxes, probe):
    """Brute-force replacement of BoxArray.intersections (boxarray.py:169)."""
    out = []
    for i, b in enumerate(boxes):
        m = meet(b, probe)
        if m is not None:
            out.append((i, m))
    return out


def fill_records(boxes, ngrow, domain, periodic):
    """_build_fill (fabarray.py:262-277): records (src, dst, src_box, shift)."""
    e = ext(domain)
    for d in range(len(e)):
        if periodic[d] and ngrow > e[d]:
            raise ValueError("ghost width exceeds domain extent in a periodic dimension")
    shifts = periodic_shifts(domain, periodic)
    zero = tuple(0 for _ in e)
    recs = []
    for j, valid in enumerate(boxes):
        if ngrow == 0:
            continue
        for piece in box_diff(grow(valid, ngrow), valid):
            for s in shifts:
                for i, ov in _overlaps(boxes, shift(piece, tuple(-x for x in s))):
                    if i == j and s == zero:
                        continue
                    recs.append((i, j, ov, s))
    return _sort(recs)


def copy_records(dst_boxes, src_boxes, dst_ngrow=0, domain=None, periodic=None):
    """_build_copy (fabarray.py:291-302) / build_plan_copy_grown (coarse_fine.py:201-220)."""
    dim = len(dst_boxes[0][0]) if dst_boxes else 3
    shifts = [tuple([0] * dim)] if domain is None else periodic_shifts(domain, periodic or (False,) * dim)
    recs = []
    for j, b in enumerate(dst_boxes):
        target = grow(b, dst_ngrow)
        for s in shifts:
            for i, ov in _overlaps(src_boxes, shift(target, tuple(-x for x in s))):
                recs.append((i, j, ov, s))
    return _sort(recs)


def sum_records(boxes, ngrow, domain, periodic):
    """build_plan_sum_boundary (fabarray.py:305-318): the fill plan transposed."""
    out = []
    for i, j, ov, s in fill_records(boxes, ngrow, domain, periodic):
        out.append((j, i, shift(ov, s), tuple(-x for x in s)))
    return _sort(out)


def records_table(recs):
    """int32 (n, 11) table in the device library's 3-D padded layout."""
    t = np.zeros((len(recs), 11), dtype=np.int32)
    for r, (i, j, ov, s) in enumerate(recs):
        dim = len(s)
        pad = 3 - dim
        t[r, 0] = i
        t[r, 1] = j
        t[r, 2 + pad : 5] = ov[0]
        t[r, 5 + pad : 8] = ov[1]
        t[r, 8 + pad : 11] = s
    return t


# ---------------------------------------------------------------------------
# storage + executor (fabarray.py:28-66, 326-406)
# ---------------------------------------------------------------------------


def make_fabs(boxes, ncomp, ngrow, fill=0.0):
    return {i: np.full((ncomp,) + tuple(e + 2 * ngrow for e in ext(b)), fill) for i, b in enumerate(boxes)}


def region_index(box, ngrow, region):
    glo = tuple(x - ngrow for x in box[0])
    return tuple(slice(region[0][d] - glo[d], region[1][d] - glo[d] + 1) for d in range(len(glo)))


def execute(recs, src_boxes, src_fabs, src_ngrow, dst_boxes, dst_fabs, dst_ngrow, add=False):
    """Two-phase: stage every source slice, then apply in plan order
    (_execute_plan, fabarray.py:326-361; rank grouping does not change results)."""
    staged = [src_fabs[i][(slice(None),) + region_index(src_boxes[i], src_ngrow, ov)].copy() for i, _, ov, _ in recs]
    for (i, j, ov, s), v in zip(recs, staged):
        idx = (slice(None),) + region_index(dst_boxes[j], dst_ngrow, shift(ov, s))
        if add:
            dst_fabs[j][idx] += v
        else:
            dst_fabs[j][idx] = v


def fill_boundary(boxes, fabs, ngrow, domain, periodic, width=None):
    """fabarray.py:364-374 (width < ngrow: AMReX FillBoundary(nghost))."""
    w = ngrow if width is None else width
    if w == 0:
        return
    execute(fill_records(boxes, w, domain, periodic), boxes, fabs, ngrow, boxes, fabs, ngrow)


def parallel_copy(dst_boxes, dst_fabs, dst_ngrow, src_boxes, src_fabs, src_ngrow, domain=None, periodic=None):
    """fabarray.py:377-388."""
    execute(copy_records(dst_boxes, src_boxes, 0, domain, periodic), src_boxes, src_fabs, src_ngrow, dst_boxes,
            dst_fabs, dst_ngrow)


def sum_boundary(boxes, fabs, ngrow, domain, periodic):
    """fabarray.py:391-406: fold ghosts onto valid cells in plan order, zero ghosts."""
    if ngrow == 0:
        return
    execute(sum_records(boxes, ngrow, domain, periodic), boxes, fabs, ngrow, boxes, fabs, ngrow, add=True)
    for i, b in enumerate(boxes):
        keep = fabs[i][(slice(None),) + region_index(b, ngrow, b)].copy()
        fabs[i][...] = 0
        fabs[i][(slice(None),) + region_index(b, ngrow, b)] = keep


def valid(boxes, fabs, ngrow, i, comp=None):
    v = fabs[i][(slice(None),) + region_index(boxes[i], ngrow, boxes[i])]
    return v if comp is None else v[comp]


def reduce(boxes, fabs, ngrow, kind, comp, owner=None, nranks=1):
    """fabarray.py:409-440: per-box numpy reduction, per-rank fold in box order,
    rank-0 fold in rank order."""
    local, pair = {"sum": (np.sum, np.add), "min": (np.min, np.minimum), "max": (np.max, np.maximum)}[kind]
    ident = {"sum": 0.0, "min": np.inf, "max": -np.inf}[kind]
    owner = owner or [0] * len(boxes)
    parts = []
    for r in range(nranks):
        acc = ident
        for i in range(len(boxes)):
            if owner[i] == r:
                acc = pair(acc, local(valid(boxes, fabs, ngrow, i, comp)))
        parts.append(acc)
    tot = parts[0]
    for p in parts[1:]:
        tot = pair(tot, p)
    return float(tot)


def gather(boxes, fabs, ngrow, region, comp=0, default=0.0):
    """gather_global (fabarray.py:443-455)."""
    out = np.full(ext(region), default)
    for i, b in enumerate(boxes):
        m = meet(b, region)
        if m is None:
            continue
        idx = tuple(slice(m[0][d] - region[0][d], m[1][d] - region[0][d] + 1) for d in range(len(m[0])))
        out[idx] = fabs[i][(comp,) + region_index(b, ngrow, m)]
    return out


def load_global(boxes, fabs, ngrow, domain, g):
    """conftest.fill_from_global (tests/conftest.py:45-53)."""
    for i, b in enumerate(boxes):
        sel = tuple(slice(b[0][d] - domain[0][d], b[1][d] - domain[0][d] + 1) for d in range(len(b[0])))
        fabs[i][(slice(None),) + region_index(b, ngrow, b)] = g[(slice(None),) + sel]


# ---------------------------------------------------------------------------
# inter-level (coarse_fine.py:136-185)
# ---------------------------------------------------------------------------


def coarsen_box(b, r):
    return (tuple(x // q for x, q in zip(b[0], r)), tuple(x // q for x, q in zip(b[1], r)))


def restrict_box(fine_valid, r, mode="average"):
    """Per-box restriction of average_down (coarse_fine.py:150-162)."""
    nc = fine_valid.shape[0]
    dim = fine_valid.ndim - 1
    if mode == "injection":
        return fine_valid[(slice(None),) + tuple(slice(0, None, r[d]) for d in range(dim))].copy()
    shape = [nc]
    for d in range(dim):
        shape += [fine_valid.shape[1 + d] // r[d], r[d]]
    return fine_valid.reshape(shape).mean(axis=tuple(2 + 2 * d for d in range(dim)))


def average_down(fine_boxes, fine_fabs, fine_ngrow, crse_boxes, crse_fabs, crse_ngrow, r, mode="average"):
    """average_down (coarse_fine.py:136-163): restrict onto the coarsened fine
    layout, then parallel_copy onto the coarse layout."""
    cboxes = [coarsen_box(b, r) for b in fine_boxes]
    tmp = {i: restrict_box(valid(fine_boxes, fine_fabs, fine_ngrow, i), r, mode) for i in range(len(fine_boxes))}
    parallel_copy(crse_boxes, crse_fabs, crse_ngrow, cboxes, tmp, 0)


def interp_pc(fine_boxes, fine_fabs, fine_ngrow, crse_boxes, crse_fabs, crse_ngrow, r, add=False):
    """interp_to_fine(..., 'pc') (coarse_fine.py:166-185, interp_block :60-72);
    add=True adds the interpolant (MLMG prolongation)."""
    cboxes = [coarsen_box(b, r) for b in fine_boxes]
    stage = make_fabs(cboxes, crse_fabs[0].shape[0], 0, np.nan)
    execute(copy_records(cboxes, crse_boxes, 0), crse_boxes, crse_fabs, crse_ngrow, cboxes, stage, 0)
    for i in range(len(fine_boxes)):
        blk = stage[i]
        if np.isnan(blk).any():
            raise ValueError("fine region has parent cells not covered by the coarse data")
        for d in range(blk.ndim - 1):
            blk = np.repeat(blk, r[d], axis=1 + d)
        v = valid(fine_boxes, fine_fabs, fine_ngrow, i)
        if add:
            v += blk
        else:
            v[...] = blk


def apply_domain_boundary(boxes, fabs, ngrow, domain, lo_conds, hi_conds, value=0.0):
    """apply_domain_boundary (amr_core.py:111-146)."""
    dim = len(domain[0])
    for i, b in enumerate(boxes):
        f = fabs[i]
        g = grow(b, ngrow)
        for d in range(dim):
            for side, cond in (("lo", lo_conds[d]), ("hi", hi_conds[d])):
                if cond == "periodic":
                    continue
                n = g[1][d] - g[0][d] + 1
                if side == "lo":
                    width = domain[0][d] - g[0][d]
                    if width <= 0:
                        continue
                    out_s, edge_s = slice(0, width), slice(width, width + 1)
                else:
                    width = g[1][d] - domain[1][d]
                    if width <= 0:
                        continue
                    out_s, edge_s = slice(n - width, n), slice(n - width - 1, n - width)
                o = [slice(None)] * (dim + 1)
                e = [slice(None)] * (dim + 1)
                o[1 + d] = out_s
                e[1 + d] = edge_s
                if cond == "external":
                    f[tuple(o)] = value
                else:
                    f[tuple(o)] = f[tuple(e)]
