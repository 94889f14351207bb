"""Native level / field descriptors and stream plumbing for libamrb calls."""

from __future__ import annotations

import ctypes as C
import threading

import numpy as np
import torch

from ._native import check, i32p, i64p, lib, u8p

__all__ = ["NativeLevel", "NativeField", "level_of", "field_of", "stream_ptr", "dh_array"]


class _Handle:
    _destroy = None

    def __init__(self, value):
        self.handle = C.c_void_p(value)

    def __del__(self):
        h = getattr(self, "handle", None)
        if h is not None and h.value and self._destroy:
            try:
                getattr(lib(), self._destroy)(h)
            except Exception:
                pass


class NativeLevel(_Handle):
    """amrb_level: valid boxes of one BoxArray (3-D padded) + resident mask."""

    _destroy = "amrb_level_destroy"

    def __init__(self, ba, resident):
        dim = ba.dim
        pad = 3 - dim
        t = np.zeros((len(ba), 6), dtype=np.int32)
        lohi = ba.lohi()
        t[:, pad:3] = lohi[:, :dim]
        t[:, 3 + pad : 6] = lohi[:, dim:]
        self.boxes3 = t
        self.ba = ba
        self.resident = np.asarray(resident, dtype=np.uint8)
        tb, tp = i32p(t)
        rb, rp = u8p(self.resident)
        h = C.c_void_p()
        check(lib().amrb_level_create(len(ba), tp, rp, C.byref(h)))
        super().__init__(h.value)


class NativeField(_Handle):
    """amrb_field: one FabArray's storage bound to a NativeLevel."""

    _destroy = "amrb_field_destroy"

    def __init__(self, level, fa):
        self.level = level  # keep the level alive as long as the field
        tb, tp = i64p(fa.fabtab)
        h = C.c_void_p()
        check(lib().amrb_field_create(level.handle, tp, fa.ngrow, C.byref(h)))
        super().__init__(h.value)


_levels = {}
_levels_lock = threading.Lock()


def level_of(fa):
    """Shared NativeLevel for (layout, resident set, device)."""
    key = (fa.ba.uid, fa.resident.tobytes(), str(fa.device))
    with _levels_lock:
        lv = _levels.get(key)
        if lv is None:
            lv = NativeLevel(fa.ba, fa.resident)
            _levels[key] = lv
    return lv


def field_of(fa):
    f = fa._native.get("field")
    if f is None:
        f = NativeField(level_of(fa), fa)
        fa._native["field"] = f
    return f


def stream_ptr(stream=None):
    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


def dh_array(dh):
    a = (C.c_double * 3)(*[float(x) for x in dh])
    return a
