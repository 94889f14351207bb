"""Box-loop stencil operators on device MultiFabs (the MLMG building blocks).

Each function is one libamrb launch over every resident box of a level
(the ParallelFor box loop; the reference's per-box numpy loop pattern is
advect.py:143-178).  Operands are MultiFabs on the same BoxArray; ghost
cells must already be filled (fill_boundary).  Definitions (operand order,
colouring) are those of oracle/mlmg_ref.py and the results are bit-identical.
"""

from __future__ import annotations

import ctypes as C

from ._native import AMRB_ENOTSUP, check, i32p, lib
from .device import dh_array, field_of, level_of, stream_ptr

__all__ = ["laplacian", "residual", "gsrb_color", "gsrb_sweep", "gsrb_sweep_norm", "residual_restrict", "dh_of"]


def dh_of(geom):
    """1/dx^2 per axis from Geometry.cell_size (amr_core.py:37-40)."""
    return tuple(1.0 / (c * c) for c in geom.cell_size)


def _p(fa):
    return C.c_void_p(fa.storage.data_ptr())


def _same_layout(*fas):
    ba = fas[0].ba
    for f in fas:
        f.require_cuda("stencil")
        if f.ba is not ba and f.ba != ba:
            raise ValueError("operands must share one BoxArray")
        if f.dim != 3:
            raise ValueError("stencil operators are 3-D")


def laplacian(out, phi, dh):
    """out = L(phi) on valid cells (phi ghosts of width >= 1 filled)."""
    _same_layout(out, phi)
    check(lib().amrb_lap_apply(level_of(out).handle, field_of(out).handle, _p(out), field_of(phi).handle, _p(phi),
                               dh_array(dh), stream_ptr()))


def residual(r, rhs, phi, dh):
    """r = rhs - L(phi)."""
    _same_layout(r, rhs, phi)
    check(lib().amrb_residual(level_of(r).handle, field_of(r).handle, _p(r), field_of(rhs).handle, _p(rhs),
                              field_of(phi).handle, _p(phi), dh_array(dh), stream_ptr()))


def gsrb_color(phi, rhs, dh, color):
    """One in-place GSRB colour ((i+j+k+color) % 2 == 0, global indices)."""
    _same_layout(phi, rhs)
    check(lib().amrb_gsrb_color(level_of(phi).handle, field_of(phi).handle, _p(phi), field_of(rhs).handle, _p(rhs),
                                dh_array(dh), int(color), stream_ptr()))


def fixed_lohi(fixed):
    """int32[6] (global lo, hi, 3-D padded) for the sweeps' ``fixed`` argument:
    a Box, or a (lo, hi) pair with None entries for unbounded axes."""
    import numpy as np

    if fixed is None:
        return None
    arr = np.array([-(1 << 30)] * 3 + [1 << 30] * 3, dtype=np.int32)
    lo, hi = (fixed.lo, fixed.hi) if hasattr(fixed, "lo") else fixed
    pad = 3 - len(lo)
    for d in range(len(lo)):
        if lo[d] is not None:
            arr[pad + d] = lo[d]
        if hi[d] is not None:
            arr[3 + pad + d] = hi[d]
    return arr


def _push_ptr(push):
    return None if push is None else C.c_void_p(push.ptr)


def gsrb_sweep(a, b, rhs, dh, fixed=None, push=None):
    """b = one fused red+black sweep of a (a ghosts width 2, rhs ghosts width 1
    filled).  ``fixed`` = Box outside which cells are never relaxed.  ``push``
    = ghosts.push_table(b, ...): b's width-2 ghosts are written by the kernel
    (NotImplementedError, nothing launched, if the level does not take the
    streaming sweep)."""
    _same_layout(a, b, rhs)
    fa = fixed_lohi(fixed)
    fp = None if fa is None else i32p(fa)[1]
    rc = lib().amrb_gsrb_sweep(level_of(a).handle, field_of(a).handle, _p(a), field_of(b).handle, _p(b),
                               field_of(rhs).handle, _p(rhs), dh_array(dh), fp, _push_ptr(push), stream_ptr())
    del fa
    if rc == AMRB_ENOTSUP:
        raise NotImplementedError("gsrb_sweep: ghost push needs the streaming sweep")
    check(rc)


def gsrb_sweep_norm(a, b, rhs, dh, norm, fixed=None, push=None):
    """gsrb_sweep(a, b, rhs) that also max-reduces |rhs - L(a)| over the valid
    cells of ``a`` into ``norm`` (a 1-element int64/uint64 CUDA tensor holding
    the bit pattern of a non-negative double; zero it first).  Raises
    NotImplementedError (nothing launched) when the level does not take the
    streaming sweep path."""
    _same_layout(a, b, rhs)
    fa = fixed_lohi(fixed)
    fp = None if fa is None else i32p(fa)[1]
    rc = lib().amrb_gsrb_sweep_norm(level_of(a).handle, field_of(a).handle, _p(a), field_of(b).handle, _p(b),
                                    field_of(rhs).handle, _p(rhs), dh_array(dh), fp, C.c_void_p(norm.data_ptr()),
                                    _push_ptr(push), stream_ptr())
    del fa
    if rc == AMRB_ENOTSUP:
        raise NotImplementedError("gsrb_sweep_norm: level does not take the streaming sweep path")
    check(rc)


def gsrb_sweep_pull(a, b, rhs, dh, table, norm=None, transport=None):
    """gsrb_sweep (norm None) / gsrb_sweep_norm with a's width-2 ghost fill
    done inside the sweep through ``table`` (ghosts.pull_table(a, ...)): a's
    ghosts need not be current before and are after -- the same cells as
    fill_boundary(a, ngrow=2) followed by the sweep.  With a p2p ``transport``
    the launch is also the device barrier of a p2p fill.  Raises
    NotImplementedError (nothing launched) when the level does not take the
    streaming sweep path."""
    _same_layout(a, b, rhs)
    if table is None:
        raise ValueError("gsrb_sweep_pull needs a pull table (ghosts.pull_table)")
    peers = transport is not None and transport.nranks > 1 and getattr(transport, "p2p", False)
    rc = lib().amrb_gsrb_sweep_pull(
        level_of(a).handle, field_of(a).handle, _p(a), field_of(b).handle, _p(b), field_of(rhs).handle, _p(rhs),
        dh_array(dh), C.c_void_p(table.ptr),
        transport._pads.ctypes.data_as(C.POINTER(C.c_uint64)) if peers else None,
        transport.rank if peers else 0, transport.nranks if peers else 1,
        C.c_void_p(transport._epoch.data_ptr()) if peers else None,
        None if norm is None else C.c_void_p(norm.data_ptr()), stream_ptr())
    if rc == AMRB_ENOTSUP:
        raise NotImplementedError("gsrb_sweep_pull: level does not take the streaming sweep path")
    check(rc)


def gsrb_sweep_prolong(a, b, rhs, dh, crse, push=None):
    """b = one fused red+black sweep of (a + pc-interpolated crse), periodic;
    crse on the box-local coarsened layout of a (ghosts width 1), a's ghosts
    width 2, rhs's width 1.  Same bits as prolong_from(a, crse, add=True);
    fill_boundary(a, 2); gsrb_sweep(a, b, rhs), but a is left unchanged.
    Raises NotImplementedError (nothing launched) when the level does not take
    the fused TMA sweep path."""
    _same_layout(a, b, rhs)
    if len(crse.ba) != len(a.ba):
        raise ValueError("crse must live on the box-local coarsened layout")
    rc = lib().amrb_gsrb_sweep_prolong(level_of(a).handle, field_of(a).handle, _p(a), field_of(b).handle, _p(b),
                                       field_of(rhs).handle, _p(rhs), dh_array(dh), level_of(crse).handle,
                                       field_of(crse).handle, _p(crse), _push_ptr(push), stream_ptr())
    if rc == AMRB_ENOTSUP:
        raise NotImplementedError("gsrb_sweep_prolong: level does not take the fused TMA sweep path")
    check(rc)


def residual_restrict(crse, rhs, phi, dh):
    """crse (on coarsened_layout(phi.ba, 2)) = average_down(rhs - L(phi))."""
    crse.require_cuda("residual_restrict")
    if len(crse.ba) != len(phi.ba):
        raise ValueError("crse must live on the box-local coarsened layout")
    check(lib().amrb_residual_restrict(level_of(crse).handle, field_of(crse).handle, _p(crse), field_of(rhs).handle,
                                       _p(rhs), field_of(phi).handle, _p(phi), dh_array(dh), stream_ptr()))
