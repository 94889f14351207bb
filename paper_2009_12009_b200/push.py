"""Ghost push: FillBoundary fused into the kernel that produces a field
(csrc/push.cu, include/amrb.h amrb_push_*).

A PushTable holds the fill plan's records (fabarray.py:262-277) whose source
box this rank owns, bound to the destination layout on every rank.  A producer
kernel given the table and the field's per-rank base pointers stores each valid
cell it writes also into every ghost cell the plan copies it to -- locally or
over NVLink into a peer's symmetric allocation -- so after the kernel (and, on
several GPUs, a device barrier) the field's ghosts are filled exactly as
fill_boundary(fa, ..., ngrow=width) would fill them.

Measured on B200 the pushing sweep and prolongation were slower
than "kernel + copy-program fill" on the C3 levels, so the solver keeps fills
by default (MLMG(ghost_push=False)); the path is kept, tested bit-exact, for
layouts where fills dominate.
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from ._native import AMRB_ENOTSUP, check, i32p, lib
from .device import field_of, level_of, stream_ptr
from .interlevel import ratio3
from .plans import build_plan_fill_boundary

__all__ = ["PushTable", "gsrb_sweep_push", "prolong_push"]


class PushTable:
    """Push records of ``fa``'s layout for ghost width ``width``.

    ``local=True`` (or a single-rank layout) treats every box as this rank's
    (replicated levels); otherwise destinations on other ranks are reached
    through ``fa.peer_ptrs`` (symmetric memory).  ``ok`` is False when the
    layout is not supported (boxes thinner than 2*width, non-slab records)."""

    def __init__(self, fa, domain, periodic, width, rank=0, local=None):
        self.width = int(width)
        nranks = fa.dm.nranks
        self.local = bool(local) if local is not None else (nranks == 1)
        plan = build_plan_fill_boundary(fa.ba, self.width, domain, periodic)
        tab = np.ascontiguousarray(plan.table(), dtype=np.int32)
        if self.local:
            owner = np.zeros(len(fa.ba), dtype=np.int32)
            gtab, self.rank, self.nranks = fa.fabtab, 0, 1
        else:
            owner = np.ascontiguousarray(fa.dm.owner, dtype=np.int32)
            gtab, self.rank, self.nranks = fa.global_fabtab(), int(rank), nranks
        gtab = np.ascontiguousarray(gtab, dtype=np.int64)
        h = C.c_void_p()
        st = lib().amrb_push_create(
            level_of(fa).handle, len(tab), tab.ctypes.data_as(C.POINTER(C.c_int32)),
            gtab.ctypes.data_as(C.POINTER(C.c_int64)), len(fa.ba), owner.ctypes.data_as(C.POINTER(C.c_int32)),
            self.rank, self.nranks, self.width, C.byref(h))
        self.ok = st != AMRB_ENOTSUP
        if self.ok:
            check(st)
        self.handle = h if self.ok else None

    def bases(self, fa):
        if self.local:
            b = np.array([fa.storage.data_ptr()], dtype=np.uint64)
        else:
            b = np.ascontiguousarray(fa.peer_ptrs, dtype=np.uint64)
        self._keep = b
        return b.ctypes.data_as(C.POINTER(C.c_uint64)), len(b)

    def __del__(self):
        if getattr(self, "handle", None) is not None:
            try:
                lib().amrb_push_destroy(self.handle)
            except Exception:
                pass


def gsrb_sweep_push(a, b, rhs, dh, table):
    """b = fused GSRB sweep of a (like stencil.gsrb_sweep) with b's ghosts pushed."""
    from .device import dh_array

    check(
        lib().amrb_gsrb_sweep_push(
            level_of(a).handle, field_of(a).handle, C.c_void_p(a.storage.data_ptr()), field_of(b).handle,
            C.c_void_p(b.storage.data_ptr()), field_of(rhs).handle, C.c_void_p(rhs.storage.data_ptr()),
            dh_array(dh), None, table.handle, *table.bases(b), stream_ptr(),
        )
    )


def prolong_push(fine, crse, table, add=True):
    """fine (+)= pc interpolation of crse (coarsened layout), fine's ghosts pushed."""
    _, rp = i32p(ratio3((2, 2, 2)))
    check(
        lib().amrb_prolong_push(
            level_of(fine).handle, field_of(fine).handle, C.c_void_p(fine.storage.data_ptr()),
            field_of(crse).handle, C.c_void_p(crse.storage.data_ptr()), rp, 1 if add else 0, table.handle,
            *table.bases(fine), stream_ptr(),
        )
    )
