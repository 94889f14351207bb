"""Level layouts: BoxArray (+ its spatial hash) and DistributionMapping.

Behaviour mirrors the reference's layout layer:

* BoxArray -- /root/reference/pkg/src/amrkit/boxarray.py:24-213: an ordered,
  pairwise-disjoint, immutable box list whose ``uid`` is its identity for plan
  caching (:37-38); ``max_size`` cuts from each box's lo (:127-152);
  ``intersections`` goes through a hash binned at the largest box extent so a
  query of up to twice a box examines at most 3**D bins (:216-278).
* DistributionMapping / sfc_distribute / knapsack_distribute / load_stats --
  /root/reference/pkg/src/amrkit/distribution.py:19-178.  Rank == GPU here.

The box table is also kept as a contiguous int32 ``lohi`` array (lo then hi
per box) because that is what the C-ABI plan builders consume.
"""

from __future__ import annotations

import heapq
import itertools
import threading
from collections import defaultdict

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


class BoxArray:
    """Ordered, pairwise-disjoint boxes of one index type; immutable."""

    __slots__ = ("boxes", "ixtype", "uid", "_hash", "_lock", "_lohi")

    def __init__(self, boxes, ixtype=None, validate=True):
        boxes = tuple(boxes)
        if ixtype is None:
            if not boxes:
                raise ValueError("empty BoxArray needs an explicit index type")
            ixtype = boxes[0].ixtype
        for b in boxes:
            if b.ixtype != ixtype:
                raise ValueError(f"mixed index types: {b!r} vs {ixtype!r}")
            if b.is_empty():
                raise ValueError("BoxArray may not contain empty boxes")
        set_ = object.__setattr__
        set_(self, "boxes", boxes)
        set_(self, "ixtype", ixtype)
        set_(self, "uid", _next_uid())
        set_(self, "_hash", None)
        set_(self, "_lock", threading.Lock())
        set_(self, "_lohi", None)
        if validate:
            self.validate()

    def __setattr__(self, *a):
        raise AttributeError("BoxArray is immutable")

    def validate(self):
        """Raise ValueError naming the first overlapping pair, else True."""
        if len(self.boxes) > 1:
            bins = _Bins(self.boxes)
            for i, b in enumerate(self.boxes):
                for j in bins.candidates(b, count=False):
                    if j != i and self.boxes[j].intersects(b):
                        a, c = min(i, j), max(i, j)
                        raise ValueError(
                            f"boxes {a} and {c} overlap: {self.boxes[a]!r} vs {self.boxes[c]!r}"
                        )
        return True

    @property
    def dim(self):
        return self.ixtype.dim

    def __len__(self):
        return len(self.boxes)

    def __getitem__(self, i):
        return self.boxes[i]

    def __iter__(self):
        return iter(self.boxes)

    def __eq__(self, other):
        if not isinstance(other, BoxArray):
            return NotImplemented
        return self.boxes == other.boxes and self.ixtype == other.ixtype

    def __hash__(self):
        return hash((self.boxes, self.ixtype))

    def __repr__(self):
        return f"BoxArray({len(self.boxes)} boxes, type {self.ixtype!r})"

    def dump(self):
        return "\n".join(repr(b) for b in self.boxes)

    def num_cells(self):
        return sum(b.num_cells() for b in self.boxes)

    def minimal_box(self):
        if not self.boxes:
            return Box.empty(self.dim, self.ixtype)
        t = self.lohi()
        d = self.dim
        return Box(t[:, :d].min(axis=0).tolist(), t[:, d:].max(axis=0).tolist(), self.ixtype)

    def lohi(self):
        """(nboxes, 2*dim) int32 table: lo coords then hi coords per box."""
        if self._lohi is None:
            t = np.array([tuple(b.lo) + tuple(b.hi) for b in self.boxes], dtype=np.int32)
            t = t.reshape(len(self.boxes), 2 * self.dim)
            t.setflags(write=False)
            object.__setattr__(self, "_lohi", t)
        return self._lohi

    # derived layouts
    def refine(self, ratio):
        return BoxArray([b.refine(ratio) for b in self.boxes], self.ixtype, validate=False)

    def coarsen(self, ratio):
        # may create overlap; callers check coarsenable() first
        return BoxArray([b.coarsen(ratio) for b in self.boxes], self.ixtype, validate=False)

    def coarsenable(self, ratio):
        return all(b.coarsen(ratio).refine(ratio) == b for b in self.boxes)

    def convert(self, ixtype):
        return BoxArray([b.convert(ixtype) for b in self.boxes], ixtype, validate=ixtype.is_cell())

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
        return BoxArray([b for b in self.boxes if not fully_covered(b)], self.ixtype, validate=False)

    # queries
    def _bins(self):
        if self._hash is None:
            with self._lock:
                if self._hash is None:
                    object.__setattr__(self, "_hash", BoxHash(self))
        return self._hash

    def intersections(self, q):
        """[(index, overlap)] for members meeting q, via the hash."""
        if q.ixtype != self.ixtype:
            raise ValueError("index type mismatch")
        if q.is_empty() or not self.boxes:
            return []
        out = []
        for i in self._bins().candidates(q):
            ov = self.boxes[i].intersect(q)
            if not ov.is_empty():
                out.append((i, ov))
        return out

    def owner_at(self, p):
        if not self.boxes:
            return None
        for i in self._bins().candidates_at(p):
            if self.boxes[i].contains(p):
                return i
        return None

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
    """owner[i] = rank (GPU) holding box i."""

    __slots__ = ("owner", "nranks")

    def __init__(self, owner, nranks):
        owner = tuple(int(r) for r in owner)
        nranks = int(nranks)
        if nranks < 1:
            raise ValueError("nranks must be >= 1")
        bad = [r for r in owner if not 0 <= r < nranks]
        if bad:
            raise ValueError(f"owner rank {bad[0]} outside 0..{nranks - 1}")
        object.__setattr__(self, "owner", owner)
        object.__setattr__(self, "nranks", nranks)

    def __setattr__(self, *a):
        raise AttributeError("DistributionMapping is immutable")

    def __len__(self):
        return len(self.owner)

    def __getitem__(self, i):
        return self.owner[i]

    def __iter__(self):
        return iter(self.owner)

    def __eq__(self, other):
        if not isinstance(other, DistributionMapping):
            return NotImplemented
        return self.owner == other.owner and self.nranks == other.nranks

    def __hash__(self):
        return hash((self.owner, self.nranks))

    def __repr__(self):
        return f"DistributionMapping(nranks={self.nranks}, owner={list(self.owner)})"

    def owned_indices(self, rank):
        return [i for i, r in enumerate(self.owner) if r == rank]

    @staticmethod
    def single_rank(nboxes):
        return DistributionMapping([0] * nboxes, 1)


def default_costs(ba):
    """Cells per box, the standard work estimate."""
    return np.array([float(b.num_cells()) for b in ba], dtype=np.float64)


def morton_key(center, domain):
    """Bit-interleaved position; bit k of dim d -> key bit k*D + d (dim 0 lowest)."""
    center = IntVect(center) if not isinstance(center, IntVect) else center
    dim = len(center)
    nbits = 63 // dim
    key = 0
    for d in range(dim):
        c = center[d] - domain.lo[d]
        if c < 0 or c >= (1 << nbits):
            raise ValueError(
                f"coordinate {center[d]} out of key range (needs 0 <= shifted < 2^{nbits})"
            )
        k = 0
        while c:
            if c & 1:
                key |= 1 << (k * dim + d)
            c >>= 1
            k += 1
    return key


def sfc_distribute(ba, cost, nranks):
    """Morton order, then contiguous runs of ~equal cost; each rank < len(ba) gets >= 1 box."""
    nranks = int(nranks)
    if nranks < 1:
        raise ValueError("nranks must be >= 1")
    cost = np.asarray(cost, dtype=np.float64)
    if len(cost) != len(ba):
        raise ValueError("cost length must match BoxArray length")
    n = len(ba)
    dom = ba.minimal_box() if n else Box.empty(1)
    two = None
    keys = []
    for i, b in enumerate(ba):
        two = two or IntVect((2,) * b.dim)
        keys.append((morton_key((b.lo + b.hi) // two, dom), i))
    order = [i for _, i in sorted(keys)]
    owner = [0] * n
    total = float(cost.sum())
    pos = 0
    assigned = 0.0
    for rank in range(nranks):
        left = nranks - rank
        limit = (n - pos) - (left - 1)
        goal = (total - assigned) / left
        take, run = 0, 0.0
        while take < limit:
            c = cost[order[pos + take]]
            if take and run + c > goal + 1e-12:
                break
            run += c
            take += 1
        if rank == nranks - 1:
            take = n - pos
        for i in order[pos : pos + take]:
            owner[i] = rank
        pos += take
        assigned += run
    return DistributionMapping(owner, nranks)


def knapsack_distribute(cost, nranks):
    """Longest-processing-time greedy; ties to the lower rank id."""
    nranks = int(nranks)
    if nranks < 1:
        raise ValueError("nranks must be >= 1")
    cost = np.asarray(cost, dtype=np.float64)
    owner = [0] * len(cost)
    heap = [(0.0, r) for r in range(nranks)]
    for i in sorted(range(len(cost)), key=lambda i: (-cost[i], i)):
        load, rank = heapq.heappop(heap)
        owner[i] = rank
        heapq.heappush(heap, (load + float(cost[i]), rank))
    return DistributionMapping(owner, nranks)


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
