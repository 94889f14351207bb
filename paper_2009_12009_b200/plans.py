"""Communication plans: ordered copy-record tables built by libamrb.

Same records, same order and same cache keys as the reference
(/root/reference/pkg/src/amrkit/fabarray.py:169-318,
coarse_fine.py:201-220); the builders run in C++ (csrc/plan.cpp) so a
4096-box fill plan costs milliseconds.  ``CommPlan.records`` materialises
Python ``CopyRecord`` objects on demand for parity checks; the device paths
never touch them.
"""

from __future__ import annotations

import ctypes as C
import threading

import numpy as np

from . import counters
from ._native import REC_W, check, i32p, lib, u8p
from .boxes import Box, IntVect

__all__ = [
    "CopyRecord",
    "CommPlan",
    "plan_cache_clear",
    "build_plan_fill_boundary",
    "build_plan_copy",
    "build_plan_copy_grown",
    "build_plan_sum_boundary",
    "normalize_periodic",
]


class CopyRecord:
    """Congruent copy (fabarray.py:171-182): source cell c of box src_index
    lands on destination cell c + shift of box dst_index."""

    __slots__ = ("src_index", "dst_index", "src_box", "dst_box", "shift")

    def __init__(self, src_index, dst_index, src_box, dst_box, shift):
        if dst_box != src_box.shift(shift):
            raise ValueError("dst_box must be src_box shifted by shift")
        for k, v in zip(self.__slots__, (src_index, dst_index, src_box, dst_box, shift)):
            setattr(self, k, v)

    def _fields(self):
        return tuple(getattr(self, k) for k in self.__slots__)

    def sort_key(self):
        """Apply order of CommPlan (fabarray.py:182-197)."""
        return (self.dst_index, tuple(self.dst_box.lo), self.src_index, tuple(self.shift))

    def __eq__(self, other):
        return isinstance(other, CopyRecord) and self._fields() == other._fields()

    def __repr__(self):
        return f"CopyRecord({self.src_index}->{self.dst_index}, {self.src_box!r}, shift={tuple(self.shift)})"


class CommPlan:
    """Owner of one native plan; records are in apply order."""

    __slots__ = ("_handle", "dim", "kind", "_records", "_table", "__weakref__")

    def __init__(self, handle, dim, kind):
        self._handle = C.c_void_p(handle)
        self.dim = dim
        self.kind = kind
        self._records = None
        self._table = None

    @property
    def handle(self):
        return self._handle

    def __del__(self):
        h = getattr(self, "_handle", None)
        if h is not None and h.value:
            try:
                lib().amrb_plan_destroy(h)
            except Exception:
                pass

    def size(self):
        n = C.c_int64()
        cells = C.c_int64()
        check(lib().amrb_plan_size(self._handle, C.byref(n), C.byref(cells)))
        return n.value, cells.value

    def __len__(self):
        return self.size()[0]

    def table(self):
        """int32 (n, 11): src, dst, src_lo[3], src_hi[3], shift[3] (3-D padded)."""
        if self._table is None:
            n, _ = self.size()
            t = np.zeros((n, REC_W), dtype=np.int32)
            if n:
                check(lib().amrb_plan_records(self._handle, t.ctypes.data_as(C.POINTER(C.c_int32))))
            t.setflags(write=False)
            self._table = t
        return self._table

    @property
    def records(self):
        if self._records is None:
            d = self.dim
            pad = 3 - d
            recs = []
            for row in self.table().tolist():
                lo = IntVect(row[2 + pad : 5])
                hi = IntVect(row[5 + pad : 8])
                sh = IntVect(row[8 + pad : 11])
                sb = Box(lo, hi)
                recs.append(CopyRecord(row[0], row[1], sb, sb.shift(sh), sh))
            self._records = recs
        return self._records

    def pairs(self, dm_src, dm_dst):
        """{(src_rank, dst_rank): [record ids]} preserving plan order."""
        t = self.table()
        so = np.asarray(dm_src.owner, dtype=np.int64)[t[:, 0]] if len(t) else np.zeros(0, np.int64)
        do = np.asarray(dm_dst.owner, dtype=np.int64)[t[:, 1]] if len(t) else np.zeros(0, np.int64)
        groups = {}
        for rid, key in enumerate(zip(so.tolist(), do.tolist())):
            groups.setdefault(key, []).append(rid)
        return groups


_cache = {}
_cache_lock = threading.Lock()


def plan_cache_clear():
    with _cache_lock:
        _cache.clear()


def _cached(key, build):
    with _cache_lock:
        hit = _cache.get(key)
    if hit is not None:
        return hit
    plan = build()
    with _cache_lock:
        prior = _cache.get(key)
        if prior is not None:
            return prior
        _cache[key] = plan
    counters.incr("plans_built")
    return plan


def normalize_periodic(periodic, dim):
    """None / a bool / per-axis flags -> a dim-tuple of bools."""
    if periodic is None or isinstance(periodic, bool):
        return (bool(periodic),) * dim
    return tuple(map(bool, periodic))


def _domain_arr(domain):
    return np.array(tuple(domain.lo) + tuple(domain.hi), dtype=np.int32)


def _new(fn, *args):
    h = C.c_void_p()
    check(fn(*args, C.byref(h)))
    return h.value


def build_plan_fill_boundary(ba, ngrow, domain, periodic=None):
    """Ghost-fill records (fabarray.py:254-277), cached per (layout, ngrow, wrap, domain)."""
    periodic = normalize_periodic(periodic, ba.dim)
    key = ("fill", ba.uid, ngrow, periodic, domain)

    def build():
        lohi, lohi_p = i32p(ba.lohi())
        dom, dom_p = i32p(_domain_arr(domain))
        per, per_p = u8p(np.array(periodic, dtype=np.uint8))
        h = _new(lib().amrb_plan_fill_create, ba.dim, len(ba), lohi_p, int(ngrow), dom_p, per_p)
        return CommPlan(h, ba.dim, "fill")

    return _cached(key, build)


def build_plan_copy(dst_ba, src_ba, domain=None, periodic=None):
    """dst valid <- overlapping src valid (fabarray.py:280-302)."""
    if dst_ba.ixtype != src_ba.ixtype:
        raise ValueError("index type mismatch")
    periodic = normalize_periodic(periodic, dst_ba.dim)
    if any(periodic) and domain is None:
        raise ValueError("periodic copy needs the domain box")
    key = ("copy", dst_ba.uid, src_ba.uid, periodic, domain)
    return _cached(key, lambda: _build_copy(dst_ba, src_ba, 0, domain, periodic))


def build_plan_copy_grown(dst_ba, src_ba, ngrow, domain=None, periodic=None):
    """Copy that may also target dst ghost cells (coarse_fine.py:201-220)."""
    periodic = normalize_periodic(periodic, dst_ba.dim)
    key = ("copyg", dst_ba.uid, src_ba.uid, ngrow, periodic, domain)
    return _cached(key, lambda: _build_copy(dst_ba, src_ba, ngrow, domain, periodic))


def _build_copy(dst_ba, src_ba, ngrow, domain, periodic):
    d, dp = i32p(dst_ba.lohi())
    s, sp = i32p(src_ba.lohi())
    if domain is None:
        dom_p, per_p = None, None
    else:
        dom, dom_p = i32p(_domain_arr(domain))
        per, per_p = u8p(np.array(periodic, dtype=np.uint8))
    h = _new(lib().amrb_plan_copy_create, dst_ba.dim, len(dst_ba), dp, len(src_ba), sp, int(ngrow), dom_p, per_p)
    return CommPlan(h, dst_ba.dim, "copy")


def build_plan_sum_boundary(ba, ngrow, domain, periodic=None):
    """Transpose of the fill plan (fabarray.py:305-318)."""
    periodic = normalize_periodic(periodic, ba.dim)
    key = ("sum", ba.uid, ngrow, periodic, domain)

    def build():
        lohi, lohi_p = i32p(ba.lohi())
        dom, dom_p = i32p(_domain_arr(domain))
        per, per_p = u8p(np.array(periodic, dtype=np.uint8))
        h = _new(lib().amrb_plan_sum_create, ba.dim, len(ba), lohi_p, int(ngrow), dom_p, per_p)
        return CommPlan(h, ba.dim, "sum")

    return _cached(key, build)
