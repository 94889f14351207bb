"""Inter-level AMR operators and two-level subcycled advection on device
(SURVEY.md 8(f)4).

Drop-in for ``fill_patch`` / ``snapshot_valid`` / ``FluxRegister``
(/root/reference/pkg/src/amrkit/coarse_fine.py:223-472) and the stepping of
``AdvectionSolver`` (advect.py:24-47,130-188) on a FIXED two-level hierarchy
(the hierarchy's regridding -- tagging, clustering, nesting -- stays out of
scope).  All cell arithmetic runs in csrc/amr.cu with the
reference's numpy evaluation order, so fields are bit-identical to the
reference's (tests/test_gpu_amr.py against fixtures made by the reference's own
AdvectionSolver, tests/golden/make_golden.py).

Data motion reuses the copy programs (fill_boundary / copy_into /
parallel_copy / average_down); the flux register's index lists are built once
per layout on the host and applied by one launch per (operation, dimension).
"""

from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from . import counters
from ._native import check, lib
from .boxes import Box, IntVect, box_diff
from .comm import Transport, copy_into, fill_boundary, parallel_copy
from .device import field_of, level_of, stream_ptr
from .geometry import apply_domain_boundary
from .interlevel import _scratch, as_ratio, average_down, coarsened_layout
from .multifab import FabArray
from .plans import normalize_periodic

__all__ = ["snapshot_valid", "fill_patch", "FaceFluxes", "upwind_fluxes", "apply_fluxes", "FluxRegister",
           "AdvectionSolver"]


def _vp(t):
    return C.c_void_p(t.data_ptr())


def _work(fa, kind):
    """(prefix int64[nb+1], boxes int32[nb], total) over fa's resident boxes,
    cached: kind 'valid' | 'grown' | ('face', axis3)."""
    key = ("work", kind)
    w = fa._native.get(key)
    if w is None:
        pad = 3 - fa.dim
        boxes, counts = [], []
        for i in range(len(fa.ba)):
            if not fa.resident[i]:
                continue
            e = [1, 1, 1]
            for d in range(fa.dim):
                e[pad + d] = fa.ba[i].hi[d] - fa.ba[i].lo[d] + 1
                if kind == "grown":
                    e[pad + d] += 2 * fa.ngrow
            if isinstance(kind, tuple):
                e[kind[1]] += 1
            boxes.append(i)
            counts.append(fa.ncomp * e[0] * e[1] * e[2])
        prefix = np.zeros(len(counts) + 1, dtype=np.int64)
        prefix[1:] = np.cumsum(counts)
        dev = fa.device
        w = (torch.as_tensor(prefix, device=dev), torch.as_tensor(np.array(boxes, dtype=np.int32), device=dev),
             len(boxes), int(prefix[-1]))
        fa._native[key] = w
    return w


def snapshot_valid(fa, transport=None, reuse=False):
    """Ghost-free copy of fa's valid data on the same layout (coarse_fine.py:223-228):
    one box-to-same-box copy program (no messages).  reuse=True returns a
    scratch FabArray cached on fa (overwritten by the next reuse call), so its
    copy program is built once."""
    if reuse:
        out = _scratch(fa, fa.ba, 0, "snapshot")
    else:
        out = FabArray(fa.ba, fa.dm, fa.ncomp, 0, device=fa.device, replicated=fa.replicated)
    parallel_copy(out, fa, transport if transport is not None else Transport(fa.dm.nranks))
    return out


# ---------------------------------------------------------------------------
# face fluxes and the advection update
# ---------------------------------------------------------------------------


class FaceFluxes:
    """Per real dimension d, every resident box's (ncomp, extents + e_d) face
    array, C order, boxes back to back in one device tensor."""

    def __init__(self, fa):
        self.fa = fa
        self.dim = fa.dim
        pad = 3 - fa.dim
        self.axes = [pad + d for d in range(fa.dim)]
        self.data, self.off, self.off_dev = [], [], []
        for ax in self.axes:
            prefix, boxes, nb, total = _work(fa, ("face", ax))
            off = np.zeros(len(fa.ba), dtype=np.int64)
            off[boxes.cpu().numpy()] = prefix.cpu().numpy()[:-1]
            self.off.append(off)
            self.off_dev.append(torch.as_tensor(off, device=fa.device))
            self.data.append(torch.empty(max(total, 1), dtype=torch.float64, device=fa.device))

    def box(self, i, d):
        """Torch view of box i's dimension-d face array (reference layout)."""
        b = self.fa.ba[i]
        ext = [b.hi[k] - b.lo[k] + 1 + (1 if k == d else 0) for k in range(self.dim)]
        n = self.fa.ncomp * int(np.prod(ext))
        o = int(self.off[d][i])
        return self.data[d][o : o + n].view(self.fa.ncomp, *ext)


def upwind_fluxes(phi, velocity, out=None):
    """First-order upwind face fluxes of every resident box (advect.py:24-36);
    phi's first ghost layer must be filled."""
    out = out if out is not None else FaceFluxes(phi)
    lvh, fh = level_of(phi), field_of(phi)
    for d, ax in enumerate(out.axes):
        prefix, boxes, nb, total = _work(phi, ("face", ax))
        check(lib().amrb_adv_flux(lvh.handle, fh.handle, _vp(phi.storage), _vp(prefix), _vp(boxes), nb, total,
                                  _vp(out.off_dev[d]), _vp(out.data[d]), phi.ncomp, ax, float(velocity[d]),
                                  stream_ptr()))
    return out


def apply_fluxes(phi, fluxes, dt_over_dx):
    """phi -= dt/dx[d] * (F[hi] - F[lo]) for every dimension in turn (advect.py:39-47)."""
    prefix, boxes, nb, total = _work(phi, "valid")
    fl = (C.c_void_p * 3)(*[C.c_void_p(t.data_ptr()) for t in fluxes.data] + [None] * (3 - phi.dim))
    fo = (C.c_void_p * 3)(*[C.c_void_p(t.data_ptr()) for t in fluxes.off_dev] + [None] * (3 - phi.dim))
    dt = (C.c_double * 3)(*[float(x) for x in dt_over_dx] + [0.0] * (3 - phi.dim))
    check(lib().amrb_adv_update(level_of(phi).handle, field_of(phi).handle, _vp(phi.storage), _vp(prefix), _vp(boxes),
                                nb, total, fl, fo, phi.ncomp, phi.dim, dt, stream_ptr()))


def _axpby(out, a, x, b, y):
    prefix, boxes, nb, total = _work(out, "valid")
    check(lib().amrb_axpby(level_of(out).handle, _vp(prefix), _vp(boxes), nb, total, field_of(out).handle,
                           _vp(out.storage), float(a), field_of(x).handle, _vp(x.storage), float(b),
                           field_of(y).handle, _vp(y.storage), stream_ptr()))


# ---------------------------------------------------------------------------
# fill_patch
# ---------------------------------------------------------------------------


def fill_patch(dst, fine_src, crse_old, crse_new, time_weight, ratio, transport, domain=None, periodic=None,
               kind="linear", boundary=None, geom=None, check_coverage=True):
    """Fill dst (valid + ghost cells) from fine data where available, else from
    time-blended coarse data interpolated to the fine level
    (coarse_fine.py:231-309): blend (1-w)*old + w*new, copy the blend onto the
    coarsened layout with ghosts (NaN elsewhere), interpolate every grown cell
    on the device, then let fine copies win, apply physical BCs, and reject
    in-domain cells neither level covers (check_coverage=False skips that
    host-synchronising test, e.g. on a fixed hierarchy after its first fill)."""
    if not 0.0 <= time_weight <= 1.0:
        raise ValueError("time_weight must lie in [0, 1]")
    if kind not in ("linear", "pc"):
        raise ValueError(f"unknown interpolation kind {kind!r}")
    dim = dst.dim
    ratio = as_ratio(ratio, dim)
    # scratch FabArrays are cached on dst / crse_new (their copy programs are
    # built once); each is fully rewritten before use
    if fine_src is dst:
        fine_src = snapshot_valid(dst, transport, reuse=True)
    # coarse data at the fill time: an endpoint as is, else the linear blend
    # (1 - w) old + w new on the device (coarse_fine.py:248-258)
    endpoint = {0.0: crse_old, 1.0: crse_new}.get(time_weight, None if crse_old is not None else crse_new)
    blended = endpoint
    if blended is None:
        blended = _scratch(crse_new, crse_new.ba, 0, "blend")
        _axpby(blended, 1.0 - time_weight, crse_old, time_weight, crse_new)
    margin = 1 if kind == "linear" else 0
    gc = -(-dst.ngrow // max(min(tuple(ratio)), 1)) + max(margin, 1)
    cdomain = domain.coarsen(ratio) if domain is not None else None
    stage = _scratch(dst, coarsened_layout(dst.ba, ratio), gc, "fp_stage")
    stage.setval(float("nan"))
    copy_into(stage, blended, transport, include_dst_ghosts=True, domain=cdomain, periodic=periodic)
    prefix, boxes, nb, total = _work(dst, "grown")
    r3 = [1, 1, 1]
    for d in range(dim):
        r3[3 - dim + d] = int(ratio[d])
    rp = (C.c_int32 * 3)(*r3)
    check(lib().amrb_interp(level_of(dst).handle, field_of(dst).handle, _vp(dst.storage), level_of(stage).handle,
                            field_of(stage).handle, _vp(stage.storage), _vp(prefix), _vp(boxes), nb, total,
                            dst.ncomp, dim, rp, 1 if kind == "linear" else 0, stream_ptr()))
    if fine_src is not None:
        copy_into(dst, fine_src, transport, include_dst_ghosts=True, domain=domain, periodic=periodic)
    if boundary is not None:
        apply_domain_boundary(dst, geom, boundary)
    if domain is not None and check_coverage:
        _check_covered(dst, domain, periodic)


def _check_covered(dst, domain, periodic):
    per = normalize_periodic(periodic, dst.dim)
    chk = domain.grow(IntVect(dst.ngrow if per[d] else 0 for d in range(dst.dim)))
    pad = 3 - dst.dim
    regions, boxes, counts = [], [], []
    for j in range(len(dst.ba)):
        if not dst.resident[j]:
            continue
        f = dst.fab(j)
        ov = f.gbox.intersect(chk)
        if ov.is_empty():
            continue
        lo, hi = [0, 0, 0], [0, 0, 0]
        for d in range(dst.dim):
            lo[pad + d] = ov.lo[d] - f.box.lo[d]
            hi[pad + d] = ov.hi[d] - f.box.lo[d]
        regions.append(lo + hi)
        boxes.append(j)
        counts.append(dst.ncomp * ov.num_cells())
    if not boxes:
        return
    prefix = np.zeros(len(counts) + 1, dtype=np.int64)
    prefix[1:] = np.cumsum(counts)
    dev = dst.device
    pt = torch.as_tensor(prefix, device=dev)
    bt = torch.as_tensor(np.array(boxes, dtype=np.int32), device=dev)
    rt = torch.as_tensor(np.array(regions, dtype=np.int32), device=dev)
    cnt = torch.zeros(1, dtype=torch.int64, device=dev)
    check(lib().amrb_nan_count(field_of(dst).handle, _vp(dst.storage), _vp(pt), _vp(bt), len(boxes), int(prefix[-1]),
                               _vp(rt), dst.ncomp, _vp(cnt), stream_ptr()))
    if int(cnt.item()):
        for j in boxes:  # error path: name the first offending box, like the reference
            f = dst.fab(j)
            ov = f.gbox.intersect(chk)
            if torch.isnan(f.slice(ov)).any():
                raise ValueError(f"box {j}: in-domain cells coverable by neither level")


# ---------------------------------------------------------------------------
# flux register
# ---------------------------------------------------------------------------


class FluxRegister:
    """Per coarse face on the fine-level boundary: (time-averaged fine flux -
    coarse flux), coarse_fine.py:317-472.  Patches (fine box k, dim d, side)
    in the reference's order; all patches share one device tensor."""

    def __init__(self, fine_ba, ratio, ncomp=1, device=None):
        self.ratio = as_ratio(ratio, fine_ba.dim)
        self.ncomp = int(ncomp)
        if not fine_ba.coarsenable(self.ratio):
            raise ValueError("fine BoxArray is not coarsenable by the given ratio")
        if any(int(r) != 2 for r in self.ratio) and fine_ba.dim > 1:
            raise ValueError("the device flux register supports refinement ratio 2")
        self.fine_ba = fine_ba
        self.cba = coarsened_layout(fine_ba, self.ratio)
        self.dim = fine_ba.dim
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.patches = []  # (k, d, side, lo[dim], hi[dim]) face boxes at coarse resolution
        off = 0
        self.poff = []
        for k, fc in enumerate(self.cba):
            for d in range(self.dim):
                for side in ("lo", "hi"):
                    plane = fc.lo[d] if side == "lo" else fc.hi[d] + 1
                    lo, hi = list(fc.lo), list(fc.hi)
                    lo[d] = hi[d] = plane
                    self.patches.append((k, d, side, lo, hi))
                    self.poff.append(off)
                    off += self.ncomp * int(np.prod([h - l + 1 for l, h in zip(lo, hi)]))
        self.size = off
        self.data = torch.zeros(max(off, 1), dtype=torch.float64, device=self.device)
        self._cache = {}

    # patch cell (comp, face coords) -> flat register index
    def _pidx(self, p, c, X):
        k, d, side, lo, hi = self.patches[p]
        idx = c
        for a in range(self.dim):
            idx = idx * (hi[a] - lo[a] + 1) + (X[a] - lo[a])
        return self.poff[p] + idx

    def patch(self, k, d, side):
        """Torch view of one patch (reference's p['data'] shape)."""
        p = [i for i, (kk, dd, ss, _, _) in enumerate(self.patches) if (kk, dd, ss) == (k, d, side)][0]
        _, _, _, lo, hi = self.patches[p]
        ext = [h - l + 1 for l, h in zip(lo, hi)]
        n = self.ncomp * int(np.prod(ext))
        return self.data[self.poff[p] : self.poff[p] + n].view(self.ncomp, *ext)

    def zero(self):
        check(lib().amrb_zero(_vp(self.data), self.data.numel(), stream_ptr()))
        return self

    def crse_add(self, crse_fluxes, crse_ba, domain, scale=1.0):
        """reg -= scale * coarse flux on every register face; a face plane shared
        by two coarse boxes is read from the box owning its high-side cell
        (coarse_fine.py:369-392).  crse_fluxes: FaceFluxes of the coarse level."""
        key = ("crse", crse_ba.uid, tuple(domain.lo), tuple(domain.hi))
        pairs = self._cache.get(key)
        if pairs is None:
            pairs = [self._crse_pairs(crse_fluxes, crse_ba, domain, d) for d in range(self.dim)]
            self._cache[key] = pairs
        for d in range(self.dim):
            if len(pairs[d]):
                check(lib().amrb_fr_crse(_vp(pairs[d]), len(pairs[d]) // 2, _vp(self.data), _vp(crse_fluxes.data[d]),
                                         float(scale), stream_ptr()))

    def _crse_pairs(self, fl, crse_ba, domain, dd):
        out = []
        for p, (k, d, side, plo, phi) in enumerate(self.patches):
            if d != dd:
                continue
            for ci in range(len(crse_ba)):
                cbox = crse_ba[ci]
                flo = list(cbox.lo)
                fhi = list(cbox.hi)
                fhi[d] += 1  # face-typed along d
                if cbox.hi[d] != domain.hi[d]:
                    fhi[d] -= 1  # owned faces
                rlo = [max(a, b) for a, b in zip(plo, flo)]
                rhi = [min(a, b) for a, b in zip(phi, fhi)]
                if any(a > b for a, b in zip(rlo, rhi)):
                    continue
                ext_ci = [cbox.hi[a] - cbox.lo[a] + 1 + (1 if a == d else 0) for a in range(self.dim)]
                for c in range(self.ncomp):
                    for X in np.ndindex(*[h - l + 1 for l, h in zip(rlo, rhi)]):
                        Xg = [rlo[a] + X[a] for a in range(self.dim)]
                        s = c
                        for a in range(self.dim):
                            s = s * ext_ci[a] + (Xg[a] - cbox.lo[a])
                        out += [self._pidx(p, c, Xg), int(fl.off[d][ci]) + s]
        return torch.as_tensor(np.array(out, dtype=np.int64), device=self.device)

    def fine_add(self, k, fine_fluxes, scale=1.0):
        """reg += scale * spatial average of fine box k's fluxes on its faces
        (coarse_fine.py:394-426); fine_fluxes: FaceFluxes of the fine level."""
        self._fine_add(fine_fluxes, scale, (k,))

    def fine_add_all(self, fine_fluxes, scale=1.0):
        """fine_add for every fine box in one launch per dimension."""
        self._fine_add(fine_fluxes, scale, None)

    def _fine_add(self, fl, scale, which):
        key = ("fine", which)
        lists = self._cache.get(key)
        if lists is None:
            lists = self._fine_lists(fl, which)
            self._cache[key] = lists
        for d, nsrc, seq, idx in lists:
            check(lib().amrb_fr_fine(_vp(idx), len(idx) // (1 + nsrc), nsrc, seq, _vp(self.data), _vp(fl.data[d]),
                                     float(scale), stream_ptr()))

    def _fine_lists(self, fl, which):
        groups = {}
        r = [int(x) for x in self.ratio]
        for p, (k, d, side, plo, phi) in enumerate(self.patches):
            if which is not None and k not in which:
                continue
            fb = self.fine_ba[k]
            ext = [fb.hi[a] - fb.lo[a] + 1 for a in range(self.dim)]
            fext = [ext[a] + (1 if a == d else 0) for a in range(self.dim)]
            local = 0 if side == "lo" else ext[d]
            others = [a for a in range(self.dim) if a != d]
            nsrc = int(np.prod([r[a] for a in others])) if others else 1
            # numpy coalesces the two reduced axes when the last coarse plane axis has length 1
            seq = 1 if (len(others) == 2 and ext[others[1]] // r[others[1]] == 1) else 0
            rows = groups.setdefault((d, nsrc, seq), [])
            for c in range(self.ncomp):
                for Y in np.ndindex(*[ext[a] // r[a] for a in others]):
                    X = list(plo)
                    for n_, a in enumerate(others):
                        X[a] = plo[a] + Y[n_]
                    row = [self._pidx(p, c, X)]
                    subs = [()]
                    for a in others:
                        subs = [s + (m,) for s in subs for m in range(r[a])]
                    for sub in subs:
                        fx = [0] * self.dim
                        fx[d] = local
                        for n_, a in enumerate(others):
                            fx[a] = Y[n_] * r[a] + sub[n_]
                        s = c
                        for a in range(self.dim):
                            s = s * fext[a] + fx[a]
                        row.append(int(fl.off[d][k]) + s)
                    rows.extend(row)
        return [(d, nsrc, seq, torch.as_tensor(np.array(rows, dtype=np.int64), device=self.device))
                for (d, nsrc, seq), rows in sorted(groups.items())]

    def reflux(self, crse, dt_over_dx, domain, periodic=None):
        """crse (uncovered cells next to the fine region) += sign * dt/dx * reg,
        every target's contributions in patch order (coarse_fine.py:428-472)."""
        per = normalize_periodic(periodic, self.dim)
        if np.isscalar(dt_over_dx):
            dt_over_dx = [float(dt_over_dx)] * self.dim
        key = ("reflux", crse.ba.uid, tuple(domain.lo), tuple(domain.hi), per, crse.serial)
        plan = self._cache.get(key)
        if plan is None:
            plan = self._reflux_plan(crse, domain, per)
            self._cache[key] = plan
        tgt, start, src, sign, dims = plan
        if not len(tgt):
            return
        ckey = key + ("coef",) + tuple(float(x) for x in dt_over_dx)
        coef_t = self._cache.get(ckey)
        if coef_t is None:  # (sign * dt/dx[d]) per contribution, like the reference's scalar
            coef = np.array([sign[e] * float(dt_over_dx[dims[e]]) for e in range(len(sign))], dtype=np.float64)
            coef_t = torch.as_tensor(coef, device=self.device)
            self._cache[ckey] = coef_t
        check(lib().amrb_fr_reflux(_vp(tgt), _vp(start), len(tgt), _vp(src), _vp(coef_t), _vp(crse.storage),
                                   _vp(self.data), stream_ptr()))

    def _reflux_plan(self, crse, domain, per):
        ext = domain.extents()
        contrib = {}  # target element -> [(reg index, sign, d)] in patch order
        order = []
        for p, (k, d, side, plo, phi) in enumerate(self.patches):
            fc = self.cba[k]
            sign = -1.0 if side == "lo" else 1.0
            clo, chi = list(plo), list(phi)
            clo[d] = chi[d] = fc.lo[d] - 1 if side == "lo" else fc.hi[d] + 1
            adj = Box(IntVect(clo), IntVect(chi))
            shift = [0] * self.dim
            if adj.lo[d] < domain.lo[d]:
                if not per[d]:
                    continue
                shift[d] = ext[d]
            elif adj.hi[d] > domain.hi[d]:
                if not per[d]:
                    continue
                shift[d] = -ext[d]
            wrapped = adj.shift(IntVect(shift))
            for ci, ov in crse.ba.intersections(wrapped):
                pieces = [ov]
                for _, cov in self.cba.intersections(ov):
                    pieces = [q for piece in pieces for q in box_diff(piece, cov)]
                if not crse.resident[ci]:
                    continue
                f = crse.fab(ci)
                for piece in pieces:
                    for c in range(self.ncomp):
                        for Xc in piece.cells():
                            Xf = [Xc[a] - shift[a] for a in range(self.dim)]  # face region = cell - shift (+1 lo side)
                            if side == "lo":
                                Xf[d] += 1
                            t = _elem(crse, ci, c, Xc)
                            if t not in contrib:
                                contrib[t] = []
                                order.append(t)
                            contrib[t].append((self._pidx(p, c, Xf), sign, d))
            del f
        tgt, start, src, sign, dims = [], [0], [], [], []
        for t in order:
            tgt.append(t)
            for s, sg, dd in contrib[t]:
                src.append(s)
                sign.append(sg)
                dims.append(dd)
            start.append(len(src))
        dev = self.device
        return (torch.as_tensor(np.array(tgt, dtype=np.int64), device=dev),
                torch.as_tensor(np.array(start, dtype=np.int64), device=dev),
                torch.as_tensor(np.array(src, dtype=np.int64), device=dev), sign, dims)


def _elem(fa, i, c, X):
    """Element offset of cell X (global) comp c of box i in fa's storage."""
    t = fa.fabtab[i]
    pad = 3 - fa.dim
    x3 = [0, 0, 0]
    for d in range(fa.dim):
        x3[pad + d] = X[d]
    return int(t[0] + c * t[1] + (x3[0] - t[4]) * t[2] + (x3[1] - t[5]) * t[3] + (x3[2] - t[6]))


# ---------------------------------------------------------------------------
# two-level subcycled advection (advect.py:130-188) on a fixed hierarchy
# ---------------------------------------------------------------------------


class AdvectionSolver:
    """Two-level conservative upwind advection with subcycling, average-down
    and refluxing, every cell operation on the device.  The hierarchy (ba0,
    dm0, ba1, dm1) is given -- regridding is out of scope.

    ``AdvectionSolver(geom0, ba0, dm0, ba1, dm1, ratio, velocity, cfl=0.45,
    use_reflux=True)``; fields ``phi[0]``, ``phi[1]`` (ncomp 1, ngrow 1);
    ``step()`` returns dt like the reference."""

    def __init__(self, geom0, ba0, dm0, ba1, dm1, ratio, velocity, cfl=0.45, use_reflux=True, transport=None,
                 use_graph=True):
        self.geoms = [geom0, geom0.refine(as_ratio(ratio, geom0.dim))]
        self.ratio = as_ratio(ratio, geom0.dim)
        self.velocity = tuple(float(v) for v in velocity)
        self.cfl = float(cfl)
        self.use_reflux = bool(use_reflux)
        self.transport = transport if transport is not None else Transport(dm0.nranks)
        self.phi = [FabArray(ba0, dm0, 1, 1), FabArray(ba1, dm1, 1, 1)]
        self.fluxreg = FluxRegister(ba1, self.ratio, 1, device=self.phi[0].device)
        self._cf = FaceFluxes(self.phi[0])
        self._ff = FaceFluxes(self.phi[1])
        self.time = 0.0
        self.step_count = 0
        self.use_graph = use_graph
        self._graph = None
        self._dt = None

    @property
    def dim(self):
        return self.geoms[0].dim

    def dt_coarse(self):
        g = self.geoms[0]
        speed = sum(abs(self.velocity[d]) / g.cell_size[d] for d in range(self.dim))
        return self.cfl / speed if speed > 0 else 1.0

    def step(self):
        """One coarse step.  The first two run eagerly (the first also checks
        that both levels cover every fine ghost cell); later steps replay a
        CUDA graph of the identical launch sequence (dt, the hierarchy and
        every buffer are fixed)."""
        dt = self.dt_coarse()
        if self._graph is not None:
            self._graph.replay()
            self._replay_counts()
        elif self.use_graph and self.step_count >= 2:
            g = torch.cuda.CUDAGraph()
            s = torch.cuda.Stream()
            s.wait_stream(torch.cuda.current_stream())
            # the step's message / byte tallies are accounted on the host while
            # the launches are captured; a replay adds the same amounts
            # (counters.py names, transport.py:40-58 counts per step)
            before = counters.snapshot()
            # NCCL send/recv inside a capture need the relaxed mode
            mode = "relaxed" if self.transport.mode == "nccl" else "global"
            with torch.cuda.stream(s):
                with torch.cuda.graph(g, stream=s, capture_error_mode=mode):
                    self._advance(dt, check=False)
            torch.cuda.current_stream().wait_stream(s)
            after = counters.snapshot()
            self._step_counts = {k: after[k] - before.get(k, 0) for k in ("transport_messages", "transport_bytes")
                                 if after.get(k, 0) != before.get(k, 0)}
            self._graph = g
            g.replay()  # capture records the launches without running them
        else:
            self._advance(dt, check=self.step_count == 0)
        self.time += dt
        self.step_count += 1
        return dt

    def _replay_counts(self):
        for k, v in getattr(self, "_step_counts", {}).items():
            counters.incr(k, v)

    def _advance(self, dt, check):
        dim = self.dim
        gc, gf = self.geoms
        phi_c, phi_f = self.phi
        crse_old = snapshot_valid(phi_c, self.transport, reuse=True)
        dto_dx_c = [dt / gc.cell_size[d] for d in range(dim)]
        fill_boundary(phi_c, self.transport, gc.domain, gc.periodic)
        upwind_fluxes(phi_c, self.velocity, self._cf)
        apply_fluxes(phi_c, self._cf, dto_dx_c)
        self.fluxreg.zero()
        self.fluxreg.crse_add(self._cf, phi_c.ba, gc.domain, scale=1.0)
        nsub = max(tuple(self.ratio))
        dt_f = dt / nsub
        dto_dx_f = [dt_f / gf.cell_size[d] for d in range(dim)]
        for m in range(nsub):
            fill_patch(phi_f, phi_f, crse_old, phi_c, time_weight=m / nsub, ratio=self.ratio,
                       transport=self.transport, domain=gf.domain, periodic=gf.periodic, kind="linear",
                       check_coverage=check)
            upwind_fluxes(phi_f, self.velocity, self._ff)
            apply_fluxes(phi_f, self._ff, dto_dx_f)
            self.fluxreg.fine_add_all(self._ff, scale=1.0 / nsub)
        average_down(phi_f, phi_c, self.ratio, self.transport)
        if self.use_reflux:
            self.fluxreg.reflux(phi_c, dto_dx_c, gc.domain, gc.periodic)

    def total_mass(self):
        """Volume-weighted composite sum (advect.py:202-225), evaluated like the
        reference (per-box numpy sums) on a host copy."""
        total = 0.0
        for lev in range(2):
            vol = float(np.prod(self.geoms[lev].cell_size))
            fa = self.phi[lev]
            cover = coarsened_layout(self.phi[1].ba, self.ratio) if lev == 0 else None
            s = 0.0
            for i in range(len(fa.ba)):
                arr = fa.fab(i).valid(0).cpu().numpy()
                s += float(arr.sum())
                if cover is not None:
                    b = fa.ba[i]
                    for _, ov in cover.intersections(b):
                        sl = tuple(slice(ov.lo[d] - b.lo[d], ov.hi[d] - b.lo[d] + 1) for d in range(fa.dim))
                        s -= float(arr[sl].sum())
            total += vol * s
        return total

