"""Ghost push tables: FillBoundary fused into the kernel that writes a field.

The fill (fabarray.py:364-374, plan _build_fill :262-277) copies, for every
box B and every ghost cell of every other box within ``width`` of B, a valid
cell of B.  On a lattice of equal boxes -- what ``max_size`` cuts and what the
MLMG's one-box-per-GPU levels are -- the destinations of B's cells depend only
on which faces a cell is near: a cell within ``width`` of B's low-x face lands
in the high-x ghost layer of the box across that face (possibly B itself
through the periodic wrap, possibly a box on another GPU), a cell near an edge
or corner also lands in the diagonal neighbours, and so on.  So one table of 26
addresses per box describes the whole fill:

    tab[b, (dx+1)*9 + (dy+1)*3 + (dz+1)] = P  such that the ghost copy of B's
    valid cell (i, j, k) (box-local) lands at  P + 8*(i*s0 + j*s1 + k)

with 0 where the direction leaves a non-periodic domain (those ghosts hold
the boundary condition and are never written by a fill).  The streaming sweep
(csrc/gsrb_stream.cu) writes every output cell within ``width`` of a face also
through the table: its output's ghosts are current when the kernel ends (on
other GPUs after a device barrier) and the copy-program fill disappears.

``push_table`` returns None when the layout is not such a lattice, or when a
destination lives on another GPU whose storage is not mapped here (no
symmetric memory); callers then keep the copy-program fill.  The table is
checked against the fill plan: the cells it covers must be exactly the plan's.

``remote_only`` keeps only the destinations on other GPUs: the sweep stores
the ghost faces its peers need over NVLink while it writes them, and the
consumer's fill copies just the local-source records, as one launch that is
also the device barrier (comm.fill_boundary(_local_sources=True)).  Only the
cross-GPU part of the exchange moves into the kernel -- the part that costs a
barrier plus NVLink round trips when pulled -- and the same-GPU ghosts stay a
bulk copy (pushing those from the sweep's edge warps measured slower).
"""

from __future__ import annotations

import itertools

import numpy as np
import torch

from .multifab import world_size
from .plans import build_plan_fill_boundary, normalize_periodic

__all__ = ["PushTable", "push_table", "pull_table"]

DIRECTIONS = [d for d in itertools.product((-1, 0, 1), repeat=3) if d != (0, 0, 0)]


class PushTable:
    """Device table (int64 addresses, nboxes x 27) + whether any destination is
    on another GPU."""

    __slots__ = ("dev", "remote", "host", "width")

    def __init__(self, host, remote, width, device):
        self.host = host
        self.remote = bool(remote)
        self.width = int(width)
        self.dev = torch.as_tensor(host.reshape(-1)).to(device)

    @property
    def ptr(self):
        return self.dev.data_ptr()


def _wrap(p, domain, periodic):
    """Periodic image of point p inside domain, or None if p leaves a
    non-periodic axis."""
    out = []
    for d in range(3):
        lo, hi = domain.lo[d], domain.hi[d]
        x = p[d]
        if lo <= x <= hi:
            out.append(x)
        elif periodic[d]:
            out.append(lo + (x - lo) % (hi - lo + 1))
        else:
            return None
    return tuple(out)


def push_table(fa, domain, periodic, width=2, remote_only=False):
    """The push table of FabArray ``fa`` for ghost width ``width`` (see the
    module docstring), cached on ``fa``; None if unsupported (or, with
    ``remote_only``, when no destination is on another GPU)."""
    periodic = normalize_periodic(periodic, fa.dim)
    key = ("push", width, tuple(domain.lo), tuple(domain.hi), periodic, bool(remote_only))
    if key in fa._native:
        return fa._native[key]
    tab = _build(fa, domain, periodic, width, bool(remote_only))
    fa._native[key] = tab
    return tab


def pull_table(fa, domain, periodic, width=2):
    """The pull table of FabArray ``fa`` (csrc/gsrb_stream.cu StreamArgs::pull),
    cached on ``fa``; None if unsupported.

    tab[b, (dx+1)*9 + (dy+1)*3 + (dz+1)] = Q | remote  such that box b's ghost
    cell (i, j, k) (box-local, inside direction (dx, dy, dz)'s width-``width``
    slab) is a copy of the valid cell at  Q + 8*(i*s0 + j*s1 + k)  -- the same
    cells the fill plan copies into b's ghosts, read by the sweep itself.  Bit 0
    marks a source box on another GPU.
    """
    periodic = normalize_periodic(periodic, fa.dim)
    key = ("pull", width, tuple(domain.lo), tuple(domain.hi), periodic)
    if key in fa._native:
        return fa._native[key]
    tab = _build(fa, domain, periodic, width, pull=True)
    fa._native[key] = tab
    return tab


def _build(fa, domain, periodic, width, remote_only=False, pull=False):
    if fa.dim != 3 or fa.ncomp != 1 or fa.ngrow < width or width < 1:
        return None
    ba = fa.ba
    n = len(ba)
    if n == 0:
        return None
    ext0 = tuple(ba[0].extents())
    if any(tuple(b.extents()) != ext0 for b in ba) or min(ext0) < 2 * width:
        return None
    dist = world_size() > 1 and fa.distributed
    if dist and not fa.symmetric:
        return None  # peers' storage is not mapped here
    gtab = fa.global_fabtab() if dist else fa.fabtab
    s0, s1 = int(gtab[0][2]), int(gtab[0][3])
    if dist:
        bases = [int(x) for x in fa.peer_ptrs]
        owner = [int(r) for r in fa.dm.owner]
        me = fa.rank
    else:
        bases = [fa.storage.data_ptr()]
        owner = [0] * n
        me = 0
    g = fa.ngrow

    def origin(b):  # element offset of box b's valid lo cell in its owner's allocation
        return int(gtab[b][0]) + g * s0 + g * s1 + g

    host = np.zeros((n, 27), dtype=np.int64)
    remote = False
    covered = 0
    for b in range(n):
        if not fa.resident[b]:
            continue
        if int(fa.fabtab[b][2]) != s0 or int(fa.fabtab[b][3]) != s1:
            return None
        B = ba[b]
        if pull:
            for d in DIRECTIONS:
                probe = tuple(B.lo[a] - 1 if d[a] < 0 else (B.hi[a] + 1 if d[a] > 0 else B.lo[a]) for a in range(3))
                img = _wrap(probe, domain, periodic)
                if img is None:
                    continue  # boundary-condition ghosts: not filled
                nb = ba.owner_at(img)
                if nb is None:
                    return None
                N = ba[nb]
                if int(gtab[nb][2]) != s0 or int(gtab[nb][3]) != s1:
                    return None
                t = tuple(img[a] - probe[a] for a in range(3))
                # B's ghost slab toward d, shifted, must be N's valid cells
                g_lo = [B.lo[a] - width if d[a] < 0 else (B.hi[a] + 1 if d[a] > 0 else B.lo[a]) for a in range(3)]
                g_hi = [B.lo[a] - 1 if d[a] < 0 else (B.hi[a] + width if d[a] > 0 else B.hi[a]) for a in range(3)]
                for a in range(3):
                    lo_t, hi_t = g_lo[a] + t[a], g_hi[a] + t[a]
                    if lo_t < N.lo[a] or hi_t > N.hi[a]:
                        return None
                    if d[a] == 0 and (lo_t != N.lo[a] or hi_t != N.hi[a]):
                        return None
                covered += int(np.prod([h - l + 1 for l, h in zip(g_lo, g_hi)]))
                rel = [B.lo[a] + t[a] - N.lo[a] for a in range(3)]
                off = origin(nb) + rel[0] * s0 + rel[1] * s1 + rel[2]
                far = owner[nb] != me
                host[b, (d[0] + 1) * 9 + (d[1] + 1) * 3 + (d[2] + 1)] = (bases[owner[nb]] + 8 * off) | int(far)
                remote |= far
            continue
        for d in DIRECTIONS:
            # the first cell beyond B's d-face (inside B along axes with d = 0)
            probe = tuple(B.lo[a] - 1 if d[a] < 0 else (B.hi[a] + 1 if d[a] > 0 else B.lo[a]) for a in range(3))
            img = _wrap(probe, domain, periodic)
            if img is None:
                continue  # leaves a non-periodic face: boundary-condition ghosts
            nb = ba.owner_at(img)
            if nb is None:
                return None
            N = ba[nb]
            t = tuple(img[a] - probe[a] for a in range(3))  # periodic shift B-side -> N-side
            # B's source cells for this direction, shifted, must sit in N's ghost layer
            src_lo = [B.lo[a] if d[a] <= 0 else B.hi[a] - width + 1 for a in range(3)]
            src_hi = [B.lo[a] + width - 1 if d[a] < 0 else B.hi[a] for a in range(3)]
            for a in range(3):
                lo_t, hi_t = src_lo[a] + t[a], src_hi[a] + t[a]
                if lo_t < N.lo[a] - width or hi_t > N.hi[a] + width:
                    return None
                if d[a] != 0 and not (hi_t < N.lo[a] or lo_t > N.hi[a]):
                    return None  # would land on N's valid cells: not a lattice
                if d[a] == 0 and (lo_t != N.lo[a] or hi_t != N.hi[a]):
                    return None  # faces must match box to box
            if remote_only and owner[nb] == me:
                continue  # same-GPU ghosts: the consumer's local fill
            covered += int(np.prod([h - l + 1 for l, h in zip(src_lo, src_hi)]))
            # element offset of the destination of B's local cell (0, 0, 0)
            rel = [B.lo[a] + t[a] - N.lo[a] for a in range(3)]
            off = origin(nb) + rel[0] * s0 + rel[1] * s1 + rel[2]
            host[b, (d[0] + 1) * 9 + (d[1] + 1) * 3 + (d[2] + 1)] = bases[owner[nb]] + 8 * off
            remote |= owner[nb] != me
    # the table must cover exactly the fill plan's ghost cells of the resident boxes
    if remote_only and not remote:
        return None
    plan = build_plan_fill_boundary(ba, width, domain, periodic)
    if dist or n != int(np.count_nonzero(fa.resident)):
        table = plan.table()
        res = np.asarray(fa.resident)
        # push: records whose SOURCE box is resident here; pull: DESTINATION
        mine = res[table[:, 1 if pull else 0]]
        if remote_only:
            mine &= np.asarray(owner)[table[:, 1]] != me
        ext = table[:, 5:8] - table[:, 2:5] + 1
        want = int(np.prod(ext[mine], axis=1).sum())
    else:
        want = plan.size()[1]
    if covered != want:
        return None
    return PushTable(host, remote, width, fa.device)
