"""Geometry and physical-boundary ghost filling.

Drop-in for ``Geometry`` / ``BoundaryRecord`` / ``apply_domain_boundary``
(/root/reference/pkg/src/amrkit/amr_core.py:26-146).  ``apply_domain_boundary``
runs on the device: one launch per (axis, side) in the reference's order, so
corner cells see the same overwrite sequence.
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from ._native import check, i32p, lib
from .boxes import Box, IntVect
from .device import field_of, level_of, stream_ptr

__all__ = ["Geometry", "BoundaryRecord", "apply_domain_boundary"]


def _periodic_flags(periodic, dim):
    """None -> all False, a bool -> the same for every axis, else per axis."""
    if periodic is None or isinstance(periodic, bool):
        return (bool(periodic),) * dim
    flags = tuple(bool(p) for p in periodic)
    if len(flags) != dim:
        raise ValueError(f"periodic needs {dim} flags")
    return flags


class Geometry:
    """One level's index space mapped onto the physical box [prob_lo, prob_hi]:
    cell (lo + i) spans prob_lo + [i, i+1) * cell_size per axis, with
    cell_size = (prob_hi - prob_lo) / extent (amr_core.py:37-40, the value the
    MLMG operator's 1/dx^2 is formed from)."""

    __slots__ = ("domain", "prob_lo", "prob_hi", "cell_size", "periodic")

    def __init__(self, domain, prob_lo, prob_hi, periodic=None):
        if not domain.ixtype.is_cell():
            raise ValueError("a Geometry's domain must be cell-centred")
        lo = tuple(map(float, prob_lo))
        hi = tuple(map(float, prob_hi))
        widths = [b - a for a, b in zip(lo, hi)]
        sizes = tuple(w / n for w, n in zip(widths, domain.extents()))
        if not all(c > 0 for c in sizes):
            raise ValueError("the physical box must have positive extent on every axis")
        self.domain, self.prob_lo, self.prob_hi = domain, lo, hi
        self.cell_size = sizes
        self.periodic = _periodic_flags(periodic, domain.dim)

    @property
    def dim(self):
        return self.domain.dim

    def _with_domain(self, dom):
        return Geometry(dom, self.prob_lo, self.prob_hi, self.periodic)

    def refine(self, ratio):
        return self._with_domain(self.domain.refine(ratio))

    def coarsen(self, ratio):
        return self._with_domain(self.domain.coarsen(ratio))

    def cell_center(self, iv):
        return tuple(p0 + (i - l + 0.5) * h
                     for p0, i, l, h in zip(self.prob_lo, iv, self.domain.lo, self.cell_size))

    def cell_index(self, point):
        return IntVect(l + int(np.floor((x - p0) / h))
                       for l, x, p0, h in zip(self.domain.lo, point, self.prob_lo, self.cell_size))

    def __repr__(self):
        return f"Geometry({self.domain!r}, dx={self.cell_size}, periodic={self.periodic})"


class BoundaryRecord:
    """Physical boundary condition for each (dimension, side): 'periodic',
    'external' (ghosts take ``external_value``) or 'extrap' (ghosts copy the
    nearest in-domain plane) -- amr_core.py:73-108."""

    CONDITIONS = ("periodic", "external", "extrap")

    def __init__(self, lo, hi, external_value=0.0):
        self.lo, self.hi = tuple(lo), tuple(hi)
        bad = [c for c in self.lo + self.hi if c not in self.CONDITIONS]
        if bad:
            raise ValueError(f"unknown boundary condition {bad[0]!r}")
        self.external_value = float(external_value)

    @classmethod
    def all_periodic(cls, dim):
        return cls(["periodic"] * dim, ["periodic"] * dim)

    @classmethod
    def all_extrap(cls, dim):
        return cls(["extrap"] * dim, ["extrap"] * dim)

    def sides(self, d):
        return self.lo[d], self.hi[d]

    def check_against(self, geom):
        """The record's periodic dimensions must be the geometry's."""
        for d, want in enumerate(geom.periodic):
            says = "periodic" in self.sides(d)
            if says != want:
                raise ValueError(f"dimension {d}: the boundary record is periodic={says}, the geometry {want}")
        return True


_CODE = {"periodic": 0, "external": 1, "extrap": 2}


def apply_domain_boundary(fa, geom, record):
    """Fill ghost cells outside the physical domain per the record."""
    record.check_against(geom)
    fa.require_cuda("apply_domain_boundary")
    if fa.ngrow == 0:
        return
    dim = fa.dim
    pad = 3 - dim
    bc = np.zeros((3, 2), dtype=np.int32)
    dom = np.zeros(6, dtype=np.int32)
    for d in range(dim):
        bc[pad + d, 0] = _CODE[record.lo[d]]
        bc[pad + d, 1] = _CODE[record.hi[d]]
        dom[pad + d] = geom.domain.lo[d]
        dom[3 + pad + d] = geom.domain.hi[d]
    b, bp = i32p(bc.reshape(-1))
    dm_, dp = i32p(dom)
    check(
        lib().amrb_domain_bc(
            level_of(fa).handle,
            field_of(fa).handle,
            C.c_void_p(fa.storage.data_ptr()),
            fa.ncomp,
            dp,
            bp,
            record.external_value,
            stream_ptr(),
        )
    )
