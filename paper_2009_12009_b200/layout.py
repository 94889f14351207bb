"""Level layouts: BoxArray (+ its spatial hash) and DistributionMapping.

Behaviour mirrors the reference's layout layer:

* BoxArray -- /root/reference/pkg/src/amrkit/boxarray.py:24-213: an ordered,
  pairwise-disjoint, immutable box list whose ``uid`` is its identity for plan
  caching (:37-38); ``max_size`` cuts from each box's lo (:127-152);
  ``intersections`` goes through a hash binned at the largest box extent so a
  query of up to twice a box examines at most 3**D bins (:216-278).
* DistributionMapping / sfc_distribute / knapsack_distribute / load_stats --
  /root/reference/pkg/src/amrkit/distribution.py:19-178.  Rank == GPU here.
  The Morton keys, the SFC split and the knapsack run in libamrb
  (csrc/distribute.cpp); this module packs the box table and wraps them.

The box table is also kept as a contiguous int32 ``lohi`` array (lo then hi
per box) because that is what the C-ABI plan builders consume.
"""

from __future__ import annotations

import ctypes as C
import itertools
import threading
from collections import defaultdict
from collections.abc import Sequence

import numpy as np

from . import counters
from .boxes import Box, IndexType, IntVect, box_diff

__all__ = [
    "BoxArray",
    "BoxHash",
    "DistributionMapping",
    "default_costs",
    "morton_key",
    "sfc_distribute",
    "knapsack_distribute",
    "load_stats",
]

_uid_source = itertools.count(1)
_uid_guard = threading.Lock()


def _next_uid():
    with _uid_guard:
        return next(_uid_source)


class _Bins:
    """Uniform-grid bins over a box list; each box registered in every bin it touches."""

    __slots__ = ("dim", "size", "origin", "table")

    def __init__(self, boxes):
        self.dim = boxes[0].dim
        ext = np.array([b.extents() for b in boxes]).max(axis=0)
        org = np.array([b.lo for b in boxes]).min(axis=0)
        self.size = tuple(max(1, int(e)) for e in ext)
        self.origin = tuple(int(o) for o in org)
        self.table = defaultdict(list)
        for i, b in enumerate(boxes):
            for key in self._span(b):
                self.table[key].append(i)

    def _key(self, p):
        return tuple((p[d] - self.origin[d]) // self.size[d] for d in range(self.dim))

    def _span(self, q):
        a, b = self._key(q.lo), self._key(q.hi)
        return itertools.product(*(range(a[d], b[d] + 1) for d in range(self.dim)))

    def candidates(self, q, count=True):
        found = {}
        nbins = 0
        for key in self._span(q):
            nbins += 1
            for i in self.table.get(key, ()):
                found.setdefault(i, None)
        if count:
            counters.incr("hash_bins_examined", nbins)
            counters.incr("hash_queries")
        return list(found)

    def candidates_at(self, p):
        counters.incr("hash_bins_examined")
        counters.incr("hash_queries")
        return self.table.get(self._key(p), ())


class BoxHash(_Bins):
    """Spatial hash of a BoxArray (built lazily, cached on the array)."""

    __slots__ = ()

    def __init__(self, ba):
        if not len(ba):
            raise ValueError("cannot hash an empty BoxArray")
        super().__init__(ba.boxes)


class BoxArray(Sequence):
    """Ordered, pairwise-disjoint boxes of one index type; immutable.

    A read-only sequence of Box; ``uid`` (fresh per instance) keys the plan
    caches, equality and hashing compare the boxes and the index type."""

    __slots__ = ("boxes", "ixtype", "uid", "_hash", "_lock", "_lohi")

    def __init__(self, boxes, ixtype=None, validate=True):
        boxes = tuple(boxes)
        if ixtype is None and not boxes:
            raise ValueError("an empty BoxArray needs an explicit index type")
        ixtype = boxes[0].ixtype if ixtype is None else ixtype
        odd = next((b for b in boxes if b.ixtype != ixtype), None)
        if odd is not None:
            raise ValueError(f"mixed index types: {odd!r} vs {ixtype!r}")
        if any(b.is_empty() for b in boxes):
            raise ValueError("BoxArray may not contain empty boxes")
        init = dict(boxes=boxes, ixtype=ixtype, uid=_next_uid(), _hash=None, _lock=threading.Lock(), _lohi=None)
        for k, v in init.items():
            object.__setattr__(self, k, v)
        if validate:
            self.validate()

    def __setattr__(self, *a):
        raise AttributeError("BoxArray values cannot be modified")

    def validate(self):
        """True, or ValueError naming the first pair of overlapping boxes."""
        if len(self.boxes) < 2:
            return True
        bins = _Bins(self.boxes)
        for i, b in enumerate(self.boxes):
            clash = [j for j in bins.candidates(b, count=False) if j != i and self.boxes[j].intersects(b)]
            if clash:
                a, c = sorted((i, clash[0]))
                raise ValueError(f"boxes {a} and {c} overlap: {self.boxes[a]!r} vs {self.boxes[c]!r}")
        return True

    # -- sequence / value protocol ------------------------------------------------
    def __len__(self):
        return len(self.boxes)

    def __getitem__(self, i):
        return self.boxes[i]

    def _ident(self):
        return (self.ixtype, self.boxes)

    def __eq__(self, other):
        return self._ident() == other._ident() if isinstance(other, BoxArray) else NotImplemented

    def __hash__(self):
        return hash(self._ident())

    def __repr__(self):
        return f"BoxArray({len(self)} boxes, type {self.ixtype!r})"

    @property
    def dim(self):
        return self.ixtype.dim

    def dump(self):
        return "\n".join(map(repr, self.boxes))

    def num_cells(self):
        return int(sum(map(Box.num_cells, self.boxes)))

    def minimal_box(self):
        if len(self) == 0:
            return Box.empty(self.dim, self.ixtype)
        t, d = self.lohi(), self.dim
        return Box(t[:, :d].min(axis=0).tolist(), t[:, d:].max(axis=0).tolist(), self.ixtype)

    def lohi(self):
        """(nboxes, 2*dim) int32 table: lo coords then hi coords per box."""
        if self._lohi is None:
            t = np.array([tuple(b.lo) + tuple(b.hi) for b in self.boxes], dtype=np.int32)
            t = t.reshape(len(self.boxes), 2 * self.dim)
            t.setflags(write=False)
            object.__setattr__(self, "_lohi", t)
        return self._lohi

    # -- derived layouts (no overlap check: a coarsening may merge boxes, callers
    # test coarsenable() first; nodal layouts may share faces) ------------------
    def _each(self, fn, ixtype=None, validate=False):
        return BoxArray(list(map(fn, self.boxes)), ixtype or self.ixtype, validate=validate)

    def refine(self, ratio):
        return self._each(lambda b: b.refine(ratio))

    def coarsen(self, ratio):
        return self._each(lambda b: b.coarsen(ratio))

    def coarsenable(self, ratio):
        return all(b == b.coarsen(ratio).refine(ratio) for b in self.boxes)

    def convert(self, ixtype):
        return self._each(lambda b: b.convert(ixtype), ixtype, validate=ixtype.is_cell())

    def max_size(self, m):
        """Chop so no extent exceeds m; cuts at lo + k*m of each box, remainder last."""
        m = IntVect((m,) * self.dim) if isinstance(m, int) else IntVect(m)
        if min(m) < 1:
            raise ValueError("max_size must be >= 1 per dimension")
        out = []
        for b in self.boxes:
            cuts = [
                [(s, min(s + m[d] - 1, b.hi[d])) for s in range(b.lo[d], b.hi[d] + 1, m[d])]
                for d in range(self.dim)
            ]
            # dimension 0 outermost, matching the reference's nested chop order
            for combo in itertools.product(*cuts):
                out.append(Box([c[0] for c in combo], [c[1] for c in combo], b.ixtype))
        return BoxArray(out, self.ixtype, validate=False)

    def prune(self, fully_covered):
        return BoxArray(itertools.filterfalse(fully_covered, self.boxes), self.ixtype, validate=False)

    # -- hash-backed queries --------------------------------------------------------
    def _bins(self):
        with self._lock:  # built once, on first query
            if self._hash is None:
                object.__setattr__(self, "_hash", BoxHash(self))
            return self._hash

    def intersections(self, q):
        """[(index, overlap)] for members meeting q, via the hash."""
        if self.ixtype != q.ixtype:
            raise ValueError("index type mismatch")
        hits = [] if (q.is_empty() or not self.boxes) else self._bins().candidates(q)
        pairs = ((i, self.boxes[i].intersect(q)) for i in hits)
        return [(i, ov) for i, ov in pairs if not ov.is_empty()]

    def owner_at(self, p):
        """Index of the box holding point p, or None."""
        hits = self._bins().candidates_at(p) if self.boxes else ()
        return next((i for i in hits if self.boxes[i].contains(p)), None)

    def contains_box(self, q):
        if q.ixtype != self.ixtype:
            raise ValueError("index type mismatch")
        rest = [] if q.is_empty() else [q]
        for _, ov in self.intersections(q):
            rest = [piece for r in rest for piece in box_diff(r, ov)]
            if not rest:
                return True
        return not rest

    def complement_in(self, region):
        rest = [] if region.is_empty() else [region]
        for _, ov in self.intersections(region):
            rest = [piece for r in rest for piece in box_diff(r, ov)]
        return rest


# ---------------------------------------------------------------------------
# distribution
# ---------------------------------------------------------------------------


class DistributionMapping:
    """owner[i] = rank (GPU) holding box i; an immutable value."""

    __slots__ = ("owner", "nranks")

    def __init__(self, owner, nranks):
        nranks = int(nranks)
        if nranks < 1:
            raise ValueError("nranks must be >= 1")
        owner = tuple(map(int, owner))
        out_of_range = [r for r in owner if r < 0 or r >= nranks]
        if out_of_range:
            raise ValueError(f"owner rank {out_of_range[0]} outside 0..{nranks - 1}")
        object.__setattr__(self, "owner", owner)
        object.__setattr__(self, "nranks", nranks)

    def __setattr__(self, *a):
        raise AttributeError("DistributionMapping values cannot be modified")

    @classmethod
    def single_rank(cls, nboxes):
        return cls((0,) * nboxes, 1)

    @classmethod
    def _from_array(cls, owner, nranks):
        return cls(np.asarray(owner).tolist(), nranks)

    def owned_indices(self, rank):
        return [i for i, r in enumerate(self.owner) if r == rank]

    # sequence of owners; equality on (owner, nranks)
    def __len__(self):
        return len(self.owner)

    def __iter__(self):
        return iter(self.owner)

    def __getitem__(self, i):
        return self.owner[i]

    def __eq__(self, other):
        if isinstance(other, DistributionMapping):
            return (self.nranks, self.owner) == (other.nranks, other.owner)
        return NotImplemented

    def __hash__(self):
        return hash((self.owner, self.nranks))

    def __repr__(self):
        return f"DistributionMapping(nranks={self.nranks}, owner={list(self.owner)})"


def default_costs(ba):
    """Cells per box, the standard work estimate."""
    return np.array([float(b.num_cells()) for b in ba], dtype=np.float64)


def morton_key(center, domain):
    """Bit-interleaved curve position of an index point, shifted by domain.lo:
    bit k of axis d -> key bit k*D + d (axis 0 least significant); libamrb
    amrb_morton_key (csrc/distribute.cpp)."""
    from ._native import check, i32p, lib

    pt = [int(x) for x in center]
    key = C.c_uint64(0)
    _p, pp = i32p(pt)
    _o, op = i32p([int(x) for x in domain.lo][: len(pt)])
    check(lib().amrb_morton_key(len(pt), pp, op, C.byref(key)))
    return int(key.value)


def _checked_costs(cost, n):
    cost = np.ascontiguousarray(cost, dtype=np.float64)
    if cost.shape != (n,):
        raise ValueError("cost length must match BoxArray length")
    return cost


def sfc_distribute(ba, cost, nranks):
    """Morton order of the box centres, then contiguous runs of about equal
    cost; every rank below the box count gets at least one box
    (distribution.py:97-131; the split runs in libamrb)."""
    from ._native import check, f64p, i32p, lib

    nranks = int(nranks)
    if nranks < 1:
        raise ValueError("nranks must be >= 1")
    cost = _checked_costs(cost, len(ba))
    owner = np.zeros(len(ba), dtype=np.int32)
    if len(ba):
        _t, tp = i32p(ba.lohi())
        _c, cp = f64p(cost)
        check(lib().amrb_sfc_distribute(ba.dim, len(ba), tp, cp, float(cost.sum()), nranks,
                                        owner.ctypes.data_as(C.POINTER(C.c_int32))))
    return DistributionMapping._from_array(owner, nranks)


def knapsack_distribute(cost, nranks):
    """Longest processing time first; ties to the lower box index, then the
    lower rank (distribution.py:134-148; runs in libamrb)."""
    from ._native import check, f64p, lib

    nranks = int(nranks)
    if nranks < 1:
        raise ValueError("nranks must be >= 1")
    cost = np.ascontiguousarray(cost, dtype=np.float64).reshape(-1)
    owner = np.zeros(len(cost), dtype=np.int32)
    _c, cp = f64p(cost)
    check(lib().amrb_knapsack_distribute(len(cost), cp, nranks, owner.ctypes.data_as(C.POINTER(C.c_int32))))
    return DistributionMapping._from_array(owner, nranks)


def load_stats(dm, cost):
    """Per-rank loads and efficiency = mean/max (1.0 when idle)."""
    cost = np.asarray(cost, dtype=np.float64)
    if len(cost) != len(dm):
        raise ValueError("cost length must match mapping length")
    loads = np.zeros(dm.nranks)
    np.add.at(loads, np.asarray(dm.owner, dtype=np.int64), cost)
    mx = float(loads.max())
    mean = float(loads.mean())
    return {
        "loads": loads,
        "max_load": mx,
        "mean_load": mean,
        "efficiency": mean / mx if mx > 0 else 1.0,
    }
