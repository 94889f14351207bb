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


class Geometry:
    """Maps a level's index space to physical coordinates."""

    __slots__ = ("domain", "prob_lo", "prob_hi", "cell_size", "periodic")

    def __init__(self, domain, prob_lo, prob_hi, periodic=None):
        if not domain.ixtype.is_cell():
            raise ValueError("domain must be cell-typed")
        self.domain = domain
        self.prob_lo = tuple(float(x) for x in prob_lo)
        self.prob_hi = tuple(float(x) for x in prob_hi)
        ext = domain.extents()
        self.cell_size = tuple((h - l) / e for l, h, e in zip(self.prob_lo, self.prob_hi, ext))
        if any(cs <= 0 for cs in self.cell_size):
            raise ValueError("physical extents must be positive")
        if periodic is None:
            periodic = (False,) * domain.dim
        elif isinstance(periodic, bool):
            periodic = (periodic,) * domain.dim
        self.periodic = tuple(bool(p) for p in periodic)

    @property
    def dim(self):
        return self.domain.dim

    def refine(self, ratio):
        return Geometry(self.domain.refine(ratio), self.prob_lo, self.prob_hi, self.periodic)

    def coarsen(self, ratio):
        return Geometry(self.domain.coarsen(ratio), self.prob_lo, self.prob_hi, self.periodic)

    def cell_center(self, iv):
        return tuple(
            self.prob_lo[d] + (iv[d] - self.domain.lo[d] + 0.5) * self.cell_size[d] for d in range(self.dim)
        )

    def cell_index(self, point):
        return IntVect(
            self.domain.lo[d] + int(np.floor((point[d] - self.prob_lo[d]) / self.cell_size[d]))
            for d in range(self.dim)
        )

    def __repr__(self):
        return f"Geometry({self.domain!r}, dx={self.cell_size}, periodic={self.periodic})"


class BoundaryRecord:
    """Per (dimension, side) condition: 'periodic', 'external' (value) or 'extrap'."""

    CONDITIONS = ("periodic", "external", "extrap")

    def __init__(self, lo, hi, external_value=0.0):
        self.lo = tuple(lo)
        self.hi = tuple(hi)
        self.external_value = float(external_value)
        for c in self.lo + self.hi:
            if c not in self.CONDITIONS:
                raise ValueError(f"unknown boundary condition {c!r}")

    @staticmethod
    def all_periodic(dim):
        return BoundaryRecord(("periodic",) * dim, ("periodic",) * dim)

    @staticmethod
    def all_extrap(dim):
        return BoundaryRecord(("extrap",) * dim, ("extrap",) * dim)

    def check_against(self, geom):
        for d in range(geom.dim):
            per = self.lo[d] == "periodic" or self.hi[d] == "periodic"
            if per != geom.periodic[d]:
                raise ValueError(
                    f"dimension {d}: boundary record says periodic={per} but geometry says {geom.periodic[d]}"
                )
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
