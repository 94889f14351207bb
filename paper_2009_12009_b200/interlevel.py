"""Inter-level data motion on device: restriction and pc prolongation.

Drop-in for the reference's ``average_down`` / ``interp_to_fine(..., "pc")``
/ ``coarsened_layout`` (/root/reference/pkg/src/amrkit/coarse_fine.py:33-43,
136-185).  Same two-step structure: a box-local kernel on the coarsened fine
layout, plus a copy program onto the target layout when the layouts differ.
Only ratio 2 (or 1) per axis and the "pc" method run on the device; the MLMG
V-cycle needs nothing else.
"""

from __future__ import annotations

import ctypes as C
import threading

import numpy as np

from ._native import check, i32p, lib
from .boxes import IntVect
from .comm import copy_into, parallel_copy
from .device import field_of, level_of, stream_ptr
from .multifab import FabArray

__all__ = ["coarsened_layout", "average_down", "interp_to_fine", "as_ratio", "ratio3"]

_memo = {}
_memo_lock = threading.Lock()


def as_ratio(ratio, dim):
    if isinstance(ratio, int):
        return IntVect((ratio,) * dim)
    return ratio if isinstance(ratio, IntVect) else IntVect(ratio)


def ratio3(ratio):
    r = [1, 1, 1]
    for d, x in enumerate(ratio):
        r[3 - len(ratio) + d] = int(x)
    return np.array(r, dtype=np.int32)


def coarsened_layout(ba, ratio):
    """Memoised ba.coarsen(ratio): one stable layout (and uid) per input."""
    ratio = as_ratio(ratio, ba.dim)
    key = (ba.uid, tuple(ratio))
    with _memo_lock:
        hit = _memo.get(key)
    if hit is not None:
        return hit
    cba = ba.coarsen(ratio)
    with _memo_lock:
        return _memo.setdefault(key, cba)


def _scratch(fa, ba, ngrow, tag):
    """Per-FabArray cached scratch FabArray on another layout (same dm)."""
    key = ("scratch", tag, ba.uid, ngrow)
    s = fa._native.get(key)
    if s is None:
        s = FabArray(ba, fa.dm, fa.ncomp, ngrow, device=fa.device, replicated=fa.replicated, rank=fa.rank)
        fa._native[key] = s
    return s


def restrict_into(tmp, fine, ratio, mode=0):
    """tmp (on coarsened_layout(fine.ba)) <- restriction of fine, box-local."""
    lv = level_of(tmp)
    r, rp = i32p(ratio3(ratio))
    check(
        lib().amrb_restrict(
            lv.handle,
            field_of(tmp).handle,
            C.c_void_p(tmp.storage.data_ptr()),
            field_of(fine).handle,
            C.c_void_p(fine.storage.data_ptr()),
            fine.ncomp,
            rp,
            mode,
            stream_ptr(),
        )
    )


def prolong_from(fine, stage, ratio, add):
    """fine (+)= pc interpolation of stage (on coarsened_layout(fine.ba))."""
    lv = level_of(fine)
    r, rp = i32p(ratio3(ratio))
    check(
        lib().amrb_prolong(
            lv.handle,
            field_of(fine).handle,
            C.c_void_p(fine.storage.data_ptr()),
            field_of(stage).handle,
            C.c_void_p(stage.storage.data_ptr()),
            fine.ncomp,
            rp,
            1 if add else 0,
            stream_ptr(),
        )
    )


def average_down(fine, crse, ratio, transport, mode="average"):
    """Covered coarse cells <- mean (or injection) of their fine children."""
    ratio = as_ratio(ratio, fine.dim)
    if not fine.ba.coarsenable(ratio):
        raise ValueError("fine BoxArray is not coarsenable by the given ratio")
    if mode not in ("average", "injection"):
        raise ValueError(f"unknown restriction mode {mode!r}")
    fine.require_cuda("average_down")
    cba = coarsened_layout(fine.ba, ratio)
    if crse.ba is cba and crse.dm == fine.dm:
        restrict_into(crse, fine, ratio, 0 if mode == "average" else 1)
        return
    tmp = _scratch(fine, cba, 0, "avgdown")
    restrict_into(tmp, fine, ratio, 0 if mode == "average" else 1)
    parallel_copy(crse, tmp, transport)


def interp_to_fine(fine, crse, ratio, transport, method="pc", add=False):
    """Fill (or, with add=True, increment) fine valid cells from coarse parents."""
    ratio = as_ratio(ratio, fine.dim)
    if not fine.ba.coarsenable(ratio):
        raise ValueError("fine BoxArray is not coarsenable by the given ratio")
    if method != "pc":
        raise ValueError(f"device interpolation supports method 'pc' only, got {method!r}")
    fine.require_cuda("interp_to_fine")
    cba = coarsened_layout(fine.ba, ratio)
    if crse.ba is cba and crse.dm == fine.dm:
        prolong_from(fine, crse, ratio, add)
        return
    stage = _scratch(fine, cba, 0, "interp")
    stage.setval(float("nan"))
    copy_into(stage, crse, transport)
    if not add:
        # the reference raises when a parent cell is uncovered (coarse_fine.py:182-183)
        for f in stage.fabs.values():
            if bool(torch_isnan_any(f.valid())):
                raise ValueError("fine region has parent cells not covered by the coarse data")
    prolong_from(fine, stage, ratio, add)


def torch_isnan_any(t):
    import torch

    return torch.isnan(t).any().item()
