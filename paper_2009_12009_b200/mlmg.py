"""Geometric multigrid (MLMG) Poisson solver on device MultiFabs.

The reference has no linear solver; the algorithm is defined by
the CPU oracle (oracle/mlmg_ref.py) and this module
reproduces it bit for bit on the GPU:

* the same level hierarchy (box-local coarsening, then agglomeration onto one
  box, then single-box coarsening to the bottom);
* GSRB sweeps run as ONE fused kernel each (csrc/stencil.cu k_gsrb_sweep):
  width-2 ghost fill of the current buffer, then red (incl. the first ghost
  ring) + black in shared memory, written out of place to the level's second
  buffer -- identical to the oracle's fill/red/fill/black;
* residual + restriction are one kernel (k_resid_restrict), prolongation is
  an add kernel, the stopping norm is a deterministic device reduction;
* a whole V-cycle plus the residual norm is captured once in a CUDA graph and
  replayed per iteration (one host sync per cycle to read the norm).

Multi-GPU: one process per GPU (``Transport.distributed()``); box-local
levels exchange ghost faces by NCCL inside the copy programs; the
agglomerated levels are replicated on every rank -- each rank restricts its
boxes into a zeroed replica, an NCCL all-reduce(sum) assembles it (each cell
has exactly one non-zero contribution, so the sum is exact), and every rank
runs the identical bottom solve.  Results are bit-identical for any GPU count.
"""

from __future__ import annotations

import collections
import ctypes as C
import os

import numpy as np
import torch

from ._native import AMRB_ENOTSUP, check, i32p, lib
from .boxes import Box, IntVect
from .comm import Transport, copy_into, device_reduce, fill_boundary, parallel_copy
from .device import dh_array, field_of, level_of, stream_ptr
from .geometry import BoundaryRecord, Geometry, apply_domain_boundary
from .interlevel import coarsened_layout, prolong_from
from .layout import BoxArray, DistributionMapping
from .ghosts import pull_table, push_table
from .stencil import gsrb_sweep_prolong
from .multifab import FabArray, MultiFab, world_size

__all__ = ["MLMG", "mg_hierarchy"]


def _coarsenable(e):
    return e % 2 == 0 and e >= 8


_TAIL_MAX_EXTENT = 16  # agglomerate once the coarsened domain fits in one CTA


def mg_hierarchy(domain, ba, nranks=1, agg_cells=128**3):
    """[(domain, BoxArray, kind)] fine -> coarse.

    Same level RESOLUTIONS as oracle.mlmg_ref.mg_levels (box-local coarsening,
    agglomeration, single-box coarsening while extents are even and >= 8), but
    the device agglomerates earlier: as soon as the coarsened domain is <= 16
    cells per side (so the one-CTA coarse-tail kernel can hold the rest), and,
    with several ranks, as soon as it has <= agg_cells cells (below that a
    replicated level is cheaper than a ghost exchange per sweep).  A level's box
    decomposition does not change its values (ghost fills are exact copies),
    so results stay bit-identical to the oracle.
    """
    levels = [(domain, ba, "base")]

    def keep_boxlocal(dom):
        nxt = dom.coarsen(2)
        if max(nxt.extents()) <= _TAIL_MAX_EXTENT:
            return False
        return nranks == 1 or nxt.num_cells() > agg_cells

    while all(_coarsenable(e) for b in ba for e in b.extents()) and keep_boxlocal(domain):
        ba = coarsened_layout(ba, 2)
        domain = domain.coarsen(2)
        levels.append((domain, ba, "boxlocal"))
    if all(_coarsenable(e) for e in domain.extents()):
        domain = domain.coarsen(2)
        ba = BoxArray([domain])
        levels.append((domain, ba, "agglom"))
        while all(_coarsenable(e) for e in domain.extents()):
            domain = domain.coarsen(2)
            ba = BoxArray([domain])
            levels.append((domain, ba, "single"))
    return levels


def rebox_per_rank(ba, dm):
    """One box per rank when each rank's boxes tile a rectangle (the usual SFC
    octants / slabs), else the layout unchanged.  The solver's internal levels
    use it: fewer, larger boxes mean no inter-box ghost traffic and fills that
    touch only rank boundaries, and a level's values do not depend on how it
    is cut into boxes."""
    boxes, owners = [], []
    for r in range(dm.nranks):
        mine = [ba[i] for i in range(len(ba)) if dm[i] == r]
        if not mine:
            continue
        lo = [min(b.lo[d] for b in mine) for d in range(ba.dim)]
        hi = [max(b.hi[d] for b in mine) for d in range(ba.dim)]
        bb = Box(lo, hi)
        if bb.num_cells() != sum(b.num_cells() for b in mine):
            return ba, dm
        boxes.append(bb)
        owners.append(r)
    return BoxArray(boxes), DistributionMapping(owners, dm.nranks)


def _tail_bytes(levels):
    tot = 0
    for dom, _, _ in levels:
        e = dom.extents()
        tot += (e[0] + 2) * (e[1] + 2) * (e[2] + 2) + e[0] * e[1] * e[2]
    return 8 * tot


class _Level:
    pass


def _zero(fa):
    """Zero a FabArray's whole storage, or a device tensor (a memset node when captured)."""
    st = fa if isinstance(fa, torch.Tensor) else fa.storage
    check(lib().amrb_zero(C.c_void_p(st.data_ptr()), st.numel(), stream_ptr()))


class MLMG:
    """V(nu1, nu2) multigrid for L(phi) = rhs on a periodic 3-D domain.

    ``MLMG(geom, ba, dm, transport=None)``; ``solve(phi, rhs, rtol, max_iter)``
    takes MultiFabs on (ba, dm) and returns the final ||r||_inf; iteration count
    and history are left in ``self.iterations`` / ``self.history``.
    """

    def __init__(self, geom, ba, dm, transport=None, nu1=2, nu2=2, bottom_sweeps=32, use_graph=True,
                 ghost_push=None, agg_cells=128**3, fuse_prolong=None, cluster_tail=None,
                 grid_level_cells=None, bc=None, ghost_pull=None):
        if geom.dim != 3:
            raise ValueError("MLMG is implemented for 3-D domains")
        # boundary conditions: 'periodic' dimensions, or 'external' sides (a
        # fixed ghost value on the finest level, 0 in the coarse-level
        # correction equations) -- BoundaryRecord, amr_core.py:73-108
        if bc is None:
            if not all(geom.periodic):
                raise ValueError("a non-periodic MLMG needs a BoundaryRecord with 'external' sides")
            bc = BoundaryRecord.all_periodic(3)
        bc.check_against(geom)
        for d in range(3):
            if not geom.periodic[d] and (bc.lo[d] != "external" or bc.hi[d] != "external"):
                raise ValueError(f"MLMG supports 'periodic' and 'external' boundaries (dimension {d}: "
                                 f"{bc.lo[d]!r}/{bc.hi[d]!r})")
        self.bc = bc
        self.all_periodic = all(geom.periodic)
        self.geom = geom
        self.nu1, self.nu2, self.bottom_sweeps = int(nu1), int(nu2), int(bottom_sweeps)
        self.transport = transport if transport is not None else Transport(dm.nranks)
        if self.transport.nranks != dm.nranks:
            raise ValueError("transport rank count differs from the distribution map")
        self.dist = self.transport.mode == "nccl"
        # a captured cycle must leave every level's ping-pong buffer where it began
        self.use_graph = use_graph and self.nu1 % 2 == 0 and self.nu2 % 2 == 0 and self.bottom_sweeps % 2 == 0
        self.periodic = geom.periodic
        self.levels = []
        self.user_ba, self.user_dm = ba, dm
        ba, dm = rebox_per_rank(ba, dm)
        for dom, lba, kind in mg_hierarchy(geom.domain, ba, nranks=dm.nranks if self.dist else 1,
                                           agg_cells=agg_cells):
            lv = _Level()
            lv.index = len(self.levels)
            lv.domain, lv.ba, lv.kind = dom, lba, kind
            # cells outside [lo, hi] are never relaxed (the sweeps' ghost ring at
            # an 'external' face); unbounded along periodic axes
            lv.fixed = None if self.all_periodic else i32p(
                [dom.lo[d] if not geom.periodic[d] else -(1 << 30) for d in range(3)]
                + [dom.hi[d] if not geom.periodic[d] else (1 << 30) for d in range(3)])
            lv.replicated = kind in ("agglom", "single")
            lv.dm = dm if not lv.replicated else DistributionMapping([0], dm.nranks)
            cs = [(h - l) / e for l, h, e in zip(geom.prob_lo, geom.prob_hi, dom.extents())]
            lv.dh = tuple(1.0 / (c * c) for c in cs)
            lv.dhc = dh_array(lv.dh)
            sym = self.dist and not lv.replicated and self.transport.p2p
            mk = lambda ng: MultiFab(lba, lv.dm, 1, ng, replicated=lv.replicated, symmetric=sym)  # noqa: E731
            lv.phi = [mk(2), mk(2)]
            lv.cur = 0
            lv.rhs = mk(1)
            lv.ncells = lba.num_cells()
            self.levels.append(lv)
        # transfer scratch on the coarsened layout where the next level differs
        for l in range(len(self.levels) - 1):
            lv, nx = self.levels[l], self.levels[l + 1]
            lv.boxlocal_next = nx.kind == "boxlocal"
            if not lv.boxlocal_next:
                cba = coarsened_layout(lv.ba, 2)
                sym = self.dist and not lv.replicated and self.transport.p2p
                lv.tmp = MultiFab(cba, lv.dm, 1, 0, replicated=lv.replicated, symmetric=sym)
                lv.stage = MultiFab(cba, lv.dm, 1, 0, replicated=lv.replicated)
        # coarse tail: the longest suffix of single-box levels that fits one CTA
        n = len(self.levels)
        self.tail = n
        for t in range(n if self.all_periodic else 0):
            if all(self.levels[x].kind in ("agglom", "single") for x in range(t, n)) and _tail_bytes(
                [(self.levels[x].domain, None, None) for x in range(t, n)]
            ) <= 200 * 1024 and n - t <= 8 and t > 0:
                self.tail = t
                break
        # a 32^3 single-box level above a 16^3 .. tail joins it: the cluster
        # variant of the tail kernel (8 CTAs, the 32^3 level split in slabs
        # across their shared memory) runs it too.  cluster_tail: 0 / False
        # off, 1 / True cubic chains, 2 / None (default) also 32 x n1 x n2 top
        # levels (n1, n2 powers of two <= 32: the multi-GPU weak-scaling chains
        # 32x16x16 .. and 32x32x16 ..; at 4 GPUs the cluster tail from
        # 32x32x16 takes 47.5 us against 29 us of grid level + 35.7 us of
        # one-CTA tail, tools/r2aj.sh).  The library picks the kernel from the
        # same shape test and reports the ghost width it wrote.
        self.cluster_tail = False
        self.cluster_mode = 2 if cluster_tail is None else int(cluster_tail)
        if self.cluster_mode not in (0, 1, 2):
            raise ValueError("cluster_tail must be 0, 1, 2 or a bool")
        noncubic = self.cluster_mode == 2

        def _cl_chain(t0):
            ext = [tuple(self.levels[x].domain.extents()) for x in range(t0, n)]
            return (len(ext) >= 2 and ext[0][0] == 32 and (noncubic or all(e[0] == e[1] == e[2] for e in ext))
                    and all(2 <= e <= 32 and e & (e - 1) == 0 for es in ext for e in es)
                    and all(ext[x][d] == 2 * ext[x + 1][d] for x in range(len(ext) - 1) for d in range(3)))

        if self.cluster_mode and self.tail < n:
            t = self.tail
            if 0 < t < n and _cl_chain(t):
                self.cluster_tail = True
            elif 1 < t < n and n - t + 1 <= 8:
                top = self.levels[t - 1]
                if _cl_chain(t - 1) and len(top.ba) == 1 and (top.replicated or not self.dist):
                    self.tail = t - 1
                    self.cluster_tail = True
        # single-box levels just above the tail, small enough to be launch-
        # latency bound, run each half V-cycle as ONE grid-synchronised launch
        # (amrb_level_grid: in-place sweeps with periodic index wrap, no fills)
        # instead of ~7 fill / sweep / transfer launches
        # (grid_level_cells: largest such level, 0 = off)
        gmax = 128**3 // 2 if grid_level_cells is None else int(grid_level_cells)
        self.grid_from = self.tail
        for l in range(self.tail - 1, 0, -1) if self.tail < n and self.all_periodic else ():
            lv, nx = self.levels[l], self.levels[l + 1]
            ext = tuple(lv.domain.extents())
            if (len(lv.ba) == 1 and len(nx.ba) == 1 and (lv.replicated or not self.dist)
                    and lv.ncells <= gmax and all(e % 2 == 0 for e in ext)
                    and tuple(nx.domain.extents()) == tuple(e // 2 for e in ext)):
                self.grid_from = l
                lv.lohi_c = i32p([*lv.domain.lo, *lv.domain.hi])
            else:
                break
        if self.tail < n:
            tl = self.levels[self.tail:]
            lohi = np.zeros((len(tl), 6), dtype=np.int32)
            dhs = np.zeros((len(tl), 3), dtype=np.float64)
            for x, lv in enumerate(tl):
                lohi[x, :3] = tuple(lv.domain.lo)
                lohi[x, 3:] = tuple(lv.domain.hi)
                dhs[x] = lv.dh
            self._tail_lohi = lohi
            self._tail_dh = dhs
        # ghost push (ghosts.py): the streaming sweeps also write their
        # output's width-2 ghosts through a per-box direction table, so the
        # copy-program fill before the next consumer disappears (ghosts on
        # other GPUs: a device barrier instead).  Periodic lattice layouts.
        # Measured on one GPU (tools/mb_stream.py, C3 fine level): sweep + push
        # 88.5 us vs sweep 75 us + fill 12 us -- the ghost bytes cost the same
        # either way in a bandwidth-bound kernel, and the same-GPU j / k faces
        # are pushed by few edge warps.  ghost_push="remote" pushes only the
        # faces other GPUs need (coalesced NVLink stores from the CTAs that own
        # them); the consumer's fill then copies the same-GPU records and is the
        # device barrier -- no NVLink round trips on its critical path.  Both
        # push modes end the pushing CTAs with a system-scope fence (remote
        # stores before the consumer's barrier), which waits behind in-flight
        # PCIe copies (tools/mb_interfere.py: sweep 97 -> 263 us with the e2e
        # pipeline's copies running), and on 2 GPUs they measured 8.65 ms
        # ("remote") and 8.33 ms (True) vs 8.03 ms with p2p fills (bench.py
        # --ghost-push, tools/r2x.sh).  So the default is the fill.
        # ghost_push: None / False = fills, True = push everything, "remote".
        self.p2p = self.dist and self.transport.p2p
        if ghost_push is None:
            ghost_push = False
        if ghost_push not in (False, True, "remote"):
            raise ValueError("ghost_push must be None, False, True or 'remote'")
        if ghost_push == "remote" and not self.p2p:
            ghost_push = False  # nothing lives on another GPU
        self.ghost_push = ghost_push
        for lv in self.levels:
            lv.push = None
            if ghost_push and self.all_periodic:
                tabs = [push_table(f, lv.domain, self.periodic, 2, remote_only=ghost_push == "remote")
                        for f in lv.phi]
                if all(t is not None for t in tabs):
                    lv.push = tabs
        # ghost pull (ghosts.pull_table, csrc/gsrb_stream.cu): a sweep whose
        # input's ghosts are stale copies them itself -- every CTA the ghost
        # cells of its own footprint, before its first TMA load -- instead of
        # a copy-program fill launched before it; across GPUs the launch is
        # also the fill's device barrier, and only the CTAs that read another
        # GPU's cells wait for it.  The fill's launch, its barrier wait and its
        # NVLink round trips leave the critical path of the other CTAs.
        # Measured slower than the fills it replaces (tools/mb_pull2.py, C3 fine
        # level: sweep 75 us, fill + sweep 85 us, pull sweep 132 us; the edge
        # CTAs' copies run at loaded-HBM latency on their critical path while
        # every other CTA streams), so it is opt-in.
        # ghost_pull: None / False = fills, True = pull.
        if ghost_pull is None:
            ghost_pull = False
        self.ghost_pull = bool(ghost_pull) and not ghost_push
        for lv in self.levels:
            lv.pull = None
            if self.ghost_pull and self.all_periodic:
                tabs = [pull_table(f, lv.domain, self.periodic, 2) for f in lv.phi]
                if all(t is not None for t in tabs):
                    lv.pull = tabs
        # up-leg: prolongation fused into the first post-smoothing sweep
        # (k_gsrb_sweep5<PROL>, box-local level pairs): no separate read+write
        # pass over the fine phi and no fill after it; the restriction fills the
        # fine phi to width 2 instead of 1 and the coarse phi gets a width-1 fill
        if fuse_prolong is None:  # False: separate prolongation (A/B runs)
            fuse_prolong = True
        for l, lv in enumerate(self.levels):
            # (the fused kernel adds the parent to every tile cell, ghosts
            # included: periodic levels only)
            lv.fuse = (fuse_prolong and l < len(self.levels) - 1 and lv.boxlocal_next
                       and self.nu2 >= 1 and self.all_periodic)
        self._ghost = {}  # id(field) -> ghost width known to be current
        self._partial = set()  # fields whose cross-GPU ghosts were pushed, same-GPU ones stale
        self._pending = False  # pushes to peers since the last device barrier
        self._reads = set()  # fields whose ghosts were read since the last barrier
        top = self.levels[0]
        self.norm = torch.zeros(1, dtype=torch.float64, device=top.rhs.device)
        # the per-cycle norm reaches the host through a kernel store into pinned
        # memory (amrb_store_host): no copy-engine transfer to queue behind the
        # caller's bulk copies on other streams
        self.norm_host = torch.zeros(1, dtype=torch.float64).pin_memory()
        self.r0_dev = torch.zeros(1, dtype=torch.float64, device=top.rhs.device)
        # pinned block shared with the loop's control kernel (csrc/graph.cu):
        # rtol, (max_iter, iters), history
        # and its device twin the loop works on (nothing inside the loop touches
        # host memory): rtol, (max_iter, iters), r0, history.  Two host slots:
        # solve(wait=False) lets the caller queue the next solve before
        # reading this one's results (finish())
        self.loop_host = [torch.zeros(3 + self._HIST, dtype=torch.float64).pin_memory() for _ in range(2)]
        self._host_slot = 0
        self._queued = collections.deque()  # solves queued by solve(wait=False), oldest first
        self.loop_dev = torch.zeros(3 + self._HIST, dtype=torch.float64, device=top.rhs.device)
        self.lag = None  # decided by the first _prime()
        self._loop = None
        self.graph_replays = 0
        self.launches_per_cycle = 0
        self.iterations = 0
        self.history = []
        self.cell_updates_per_cycle = sum(
            lv.ncells * (self.nu1 + self.nu2 if i < len(self.levels) - 1 else self.bottom_sweeps)
            for i, lv in enumerate(self.levels)
        )

    # -- ghost state ---------------------------------------------------------------
    def _barrier(self):
        self.transport.peer_barrier()
        self._pending = False
        self._reads.clear()

    def _need_ghosts(self, lv, fa, width):
        """Before a kernel reads fa's ghosts (width cells)."""
        if id(fa) in self._partial:
            # peers pushed the cross-GPU ghosts (to the table's width 2): copy
            # the same-GPU ones; the launch is also the device barrier
            fill_boundary(fa, self.transport, lv.domain, self.periodic, ngrow=2, _post_barrier=False,
                          _local_sources=True)
            self._partial.discard(id(fa))
            self._ghost[id(fa)] = 2
            self._pending = False
            self._reads.clear()
        if self._ghost.get(id(fa), 0) >= width:
            if self._pending:
                self._barrier()
        else:
            self._fill(lv, fa, width)
            self._ghost[id(fa)] = width
            if self.p2p:  # the p2p fill starts with a device barrier
                self._pending = False
                self._reads.clear()
        if self.dist:
            self._reads.add(id(fa))

    def _produced(self, fa, width, pushed_to_peers=False):
        """After a kernel rewrote fa's valid cells; width = ghosts it filled."""
        self._ghost[id(fa)] = width
        self._partial.discard(id(fa))
        if pushed_to_peers:
            self._pending = True

    def _pushed(self, fa, tab):
        """After a sweep wrote fa through push table ``tab``."""
        if tab is None:
            self._produced(fa, 0)
        elif self.ghost_push == "remote":
            self._produced(fa, 0, pushed_to_peers=True)
            self._partial.add(id(fa))
        else:
            self._produced(fa, tab.width, pushed_to_peers=tab.remote)

    def _before_push(self, tab, fa):
        """Before a kernel stores into peers' ghosts of fa: no peer may still be
        reading them."""
        if tab.remote and id(fa) in self._reads:
            self._barrier()

    def _push_for(self, lv, fa):
        """The push table of lv's phi buffer fa, or None."""
        if lv.push is None:
            return None
        return lv.push[0] if fa is lv.phi[0] else lv.push[1]

    # -- building blocks ---------------------------------------------------------
    def _fill(self, lv, fa, width):
        # Inside the V-cycle a rank only rewrites cells a peer pulled after the
        # next fill's barrier (or an NCCL collective), so one barrier per fill
        # suffices for the p2p path.
        fill_boundary(fa, self.transport, lv.domain, self.periodic, ngrow=width, _post_barrier=False)
        if not self.all_periodic and lv.index > 0 and fa is not lv.rhs:
            # coarse-level homogeneous Dirichlet: ghost = -alpha_l * mirror
            # (oracle/mlmg_ref.py reflect_ghosts); the finest level's 'external'
            # ghosts are set once (set_phi) and never overwritten
            r = float(1 << lv.index)
            self._domain_bc(lv, fa, 3, -((r - 1.0) / (r + 1.0)))

    def _domain_bc(self, lv, fa, cond, value):
        bc = np.zeros((3, 2), dtype=np.int32)
        for d in range(3):
            if not self.periodic[d]:
                bc[d] = cond
        dom = np.array(list(lv.domain.lo) + list(lv.domain.hi), dtype=np.int32)
        _b, bp = i32p(bc.reshape(-1))
        _d, dp = i32p(dom)
        check(lib().amrb_domain_bc(level_of(fa).handle, field_of(fa).handle, C.c_void_p(fa.storage.data_ptr()),
                                   fa.ncomp, dp, bp, float(value), stream_ptr()))

    def _sweep(self, lv, norm=None):
        """One fused sweep lv.phi[cur] -> lv.phi[1-cur]; with ``norm`` (a
        1-element device tensor) the kernel also max-reduces |rhs - L(phi)| of
        its INPUT into it (NotImplementedError, nothing launched, where the
        level does not take the streaming kernel)."""
        a = lv.phi[lv.cur]
        b = lv.phi[1 - lv.cur]
        if lv.pull is not None and id(a) not in self._partial and self._ghost.get(id(a), 0) < 2:
            if self._sweep_pull(lv, a, b, norm):
                return
        self._need_ghosts(lv, a, 2)
        self._need_ghosts(lv, lv.rhs, 1)
        tab = self._push_for(lv, b)
        if tab is not None:
            self._before_push(tab, b)
        lvh = level_of(a)
        args = (
            lvh.handle,
            field_of(a).handle,
            C.c_void_p(a.storage.data_ptr()),
            field_of(b).handle,
            C.c_void_p(b.storage.data_ptr()),
            field_of(lv.rhs).handle,
            C.c_void_p(lv.rhs.storage.data_ptr()),
            lv.dhc,
            None if lv.fixed is None else lv.fixed[1],
        )
        push = None if tab is None else C.c_void_p(tab.ptr)
        if norm is None:
            rc = lib().amrb_gsrb_sweep(*args, push, stream_ptr())
            if rc == AMRB_ENOTSUP:  # pushing needs the streaming kernel: fill instead from now on
                lv.push, tab = None, None
                rc = lib().amrb_gsrb_sweep(*args, None, stream_ptr())
            check(rc)
        else:
            rc = lib().amrb_gsrb_sweep_norm(*args, C.c_void_p(norm.data_ptr()), push, stream_ptr())
            if rc == AMRB_ENOTSUP:
                raise NotImplementedError("level does not take the streaming sweep")
            check(rc)
        self._pushed(b, tab)
        lv.cur = 1 - lv.cur

    def _sweep_pull(self, lv, a, b, norm):
        """_sweep with the input's ghost fill done by the sweep itself
        (amrb_gsrb_sweep_pull); False (nothing launched) where the level does
        not take the streaming kernel."""
        self._need_ghosts(lv, lv.rhs, 1)
        tab = lv.pull[0] if a is lv.phi[0] else lv.pull[1]
        tr = self.transport
        peers = self.p2p
        rc = lib().amrb_gsrb_sweep_pull(
            level_of(a).handle,
            field_of(a).handle,
            C.c_void_p(a.storage.data_ptr()),
            field_of(b).handle,
            C.c_void_p(b.storage.data_ptr()),
            field_of(lv.rhs).handle,
            C.c_void_p(lv.rhs.storage.data_ptr()),
            lv.dhc,
            C.c_void_p(tab.ptr),
            tr._pads.ctypes.data_as(C.POINTER(C.c_uint64)) if peers else None,
            tr.rank if peers else 0,
            tr.nranks if peers else 1,
            C.c_void_p(tr._epoch.data_ptr()) if peers else None,
            None if norm is None else C.c_void_p(norm.data_ptr()),
            stream_ptr(),
        )
        if rc == AMRB_ENOTSUP:
            lv.pull = None
            return False
        check(rc)
        self._ghost[id(a)] = 2  # every ghost cell of a was copied by some CTA
        if peers:  # the launch was the device barrier
            self._pending = False
            self._reads.clear()
            self._reads.add(id(a))
        self._produced(b, 0)
        lv.cur = 1 - lv.cur
        return True

    def _smooth(self, lv, n):
        for _ in range(n):
            self._sweep(lv)

    def _resid_restrict(self, l):
        lv, nx = self.levels[l], self.levels[l + 1]
        phi = lv.phi[lv.cur]
        self._need_ghosts(lv, phi, 2 if lv.fuse else 1)  # the fused up-leg sweep reuses width 2
        dst = nx.rhs if lv.boxlocal_next else lv.tmp
        check(
            lib().amrb_residual_restrict(
                level_of(dst).handle,
                field_of(dst).handle,
                C.c_void_p(dst.storage.data_ptr()),
                field_of(lv.rhs).handle,
                C.c_void_p(lv.rhs.storage.data_ptr()),
                field_of(phi).handle,
                C.c_void_p(phi.storage.data_ptr()),
                lv.dhc,
                stream_ptr(),
            )
        )
        if not lv.boxlocal_next:
            self._gather_replica(lv, nx)
        self._produced(nx.rhs, 0)
        if l + 1 < self.grid_from:  # the coarse tail / grid levels read valid rhs cells only
            self._need_ghosts(nx, nx.rhs, 1)

    def _gather_replica(self, lv, nx):
        """tmp (coarsened layout of lv, maybe distributed) -> nx.rhs (one box)."""
        if self.dist and not lv.replicated and self.transport.p2p:
            # every rank pulls every rank's restricted boxes into its replica
            # over NVLink (peer-pull copy program framed by the signal barrier)
            copy_into(nx.rhs, lv.tmp, self.transport)
        elif self.dist and not lv.replicated:
            _zero(nx.rhs)
            # every rank copies its own boxes into its replica, then all-reduce(sum)
            copy_into(nx.rhs, lv.tmp, _LocalView(self.transport))
            check(
                lib().amrb_nccl_allreduce(
                    C.c_void_p(nx.rhs.storage.data_ptr()), nx.rhs.storage.numel(), 0, self.transport.nccl_comm,
                    stream_ptr(),
                )
            )
        else:
            parallel_copy(nx.rhs, lv.tmp, self.transport)

    def _prolong(self, l):
        lv, nx = self.levels[l], self.levels[l + 1]
        fine = lv.phi[lv.cur]
        crse = nx.phi[nx.cur]
        if not lv.boxlocal_next:
            tr = _LocalView(self.transport) if (self.dist and not lv.replicated) else self.transport
            copy_into(lv.stage, crse, tr)
            crse = lv.stage
        prolong_from(fine, crse, (2, 2, 2), add=True)
        self._produced(fine, 0)

    def _prolong_sweep(self, l):
        """Fused up-leg step: lv.phi <- GSRB(lv.phi + P(nx.phi)).  False (nothing
        launched) when the level does not take the fused TMA sweep path."""
        lv, nx = self.levels[l], self.levels[l + 1]
        a, b = lv.phi[lv.cur], lv.phi[1 - lv.cur]
        crse = nx.phi[nx.cur]
        self._need_ghosts(lv, a, 2)
        self._need_ghosts(lv, lv.rhs, 1)
        self._need_ghosts(nx, crse, 1)
        tab = self._push_for(lv, b)
        if tab is not None:
            self._before_push(tab, b)
        try:
            gsrb_sweep_prolong(a, b, lv.rhs, lv.dh, crse, push=tab)
        except NotImplementedError:
            lv.fuse = False
            return False
        self._pushed(b, tab)
        lv.cur = 1 - lv.cur
        return True

    def _residual_norm(self):
        top = self.levels[0]
        phi = top.phi[top.cur]
        # width 2, not 1: the next cycle's first sweep reads this phi's ghosts
        # to width 2, so one fill serves both (one fine fill less per cycle)
        self._need_ghosts(top, phi, 2)
        check(
            lib().amrb_residual_norm(
                level_of(phi).handle,
                field_of(top.rhs).handle,
                C.c_void_p(top.rhs.storage.data_ptr()),
                field_of(phi).handle,
                C.c_void_p(phi.storage.data_ptr()),
                top.dhc,
                C.c_void_p(self.norm.data_ptr()),
                stream_ptr(),
            )
        )

    def _allmax(self, t):
        if self.dist and self.transport.p2p:
            self.transport.peer_allmax(t)
        elif self.dist:
            check(lib().amrb_nccl_allreduce(C.c_void_p(t.data_ptr()), 1, 2, self.transport.nccl_comm, stream_ptr()))

    def _coarse_tail(self):
        """All tail levels in one kernel: reads rhs, writes phi of levels[tail]."""
        lv = self.levels[self.tail]
        phi = lv.phi[lv.cur]
        written = C.c_int32(0)
        lohi, lp = i32p(self._tail_lohi)
        dh = np.ascontiguousarray(self._tail_dh)
        check(
            lib().amrb_coarse_tail(
                len(self._tail_lohi),
                lp,
                dh.ctypes.data_as(C.POINTER(C.c_double)),
                field_of(lv.rhs).handle,
                C.c_void_p(lv.rhs.storage.data_ptr()),
                field_of(phi).handle,
                C.c_void_p(phi.storage.data_ptr()),
                self.nu1,
                self.nu2,
                self.bottom_sweeps,
                self.cluster_mode,
                C.byref(written),
                stream_ptr(),
            )
        )
        # ghost width the launched kernel left current (the cluster variant: 1);
        # decided by the library's own shape test, not re-derived here
        self._produced(phi, int(written.value))

    def _level_grid(self, l, up):
        """Half V-cycle of grid level l in one launch (amrb_level_grid)."""
        lv, nx = self.levels[l], self.levels[l + 1]
        phi = lv.phi[lv.cur]
        crse = nx.phi[nx.cur] if up else nx.rhs
        check(
            lib().amrb_level_grid(
                int(up),
                lv.lohi_c[1],
                lv.dhc,
                field_of(lv.rhs).handle,
                C.c_void_p(lv.rhs.storage.data_ptr()),
                field_of(phi).handle,
                C.c_void_p(phi.storage.data_ptr()),
                field_of(crse).handle,
                C.c_void_p(crse.storage.data_ptr()),
                self.nu2 if up else self.nu1,
                stream_ptr(),
            )
        )
        self._produced(phi, 1 if up else 0)
        if not up:
            self._produced(nx.rhs, 0)

    def vcycle(self, first_done=False):
        """One V(nu1, nu2) cycle; first_done: the finest level's first
        pre-smoothing sweep already ran (the previous iteration's fused
        sweep + residual norm)."""
        L = self.levels
        n = len(L)
        T = self.tail  # first level handled by the coarse-tail kernel (n: none)
        G = self.grid_from  # first grid-synchronised level (T: none)
        for l in range(G):
            lv = L[l]
            if l > 0:
                _zero(lv.phi[lv.cur])
                self._produced(lv.phi[lv.cur], 2)  # zero ghosts are the periodic fill of zero
            if l == n - 1:
                self._smooth(lv, self.bottom_sweeps)
                break
            self._smooth(lv, self.nu1 - (1 if l == 0 and first_done else 0))
            self._resid_restrict(l)
        for l in range(G, T):
            self._level_grid(l, up=False)
        if T < n:
            self._coarse_tail()
        for l in range(T - 1, G - 1, -1):
            self._level_grid(l, up=True)
        for l in range(min(G, n - 1) - 1, -1, -1):
            if L[l].fuse and self._prolong_sweep(l):
                self._smooth(L[l], self.nu2 - 1)
            else:
                self._prolong(l)
                self._smooth(L[l], self.nu2)

    # -- one solve iteration -------------------------------------------------------
    # Lagged norm (self.lag): the residual of a cycle's result is the residual of
    # the INPUT of the next cycle's first pre-smoothing sweep, which the fused
    # sweep computes from the phi / rhs it streams anyway (amrb_gsrb_sweep_norm).
    # So an iteration is "the rest of cycle n + the first sweep of cycle n+1 with
    # the norm of cycle n's result"; the sweep is out of place, so when the test
    # says stop, cycle n's solution is intact in the sweep's input buffer.  This
    # removes the separate residual-norm pass over the finest level (16 N bytes
    # per cycle).  Without the streaming sweep (or nu1 == 0) the iteration is the
    # whole cycle followed by the residual-norm kernel.
    def _body(self):
        if self.lag:
            self.vcycle(first_done=True)
            self._sweep(self.levels[0], norm=self.norm)
        else:
            self.vcycle()
            self._residual_norm()
        self._allmax(self.norm)

    def _solution_index(self):
        top = self.levels[0]
        return 1 - top.cur if self.lag else top.cur

    def _prime(self):
        """Before the first iteration: the lagged scheme runs the first
        pre-smoothing sweep of cycle 1 (its norm, of phi0, is discarded).  The
        first call decides whether the finest level takes the fused sweep +
        norm kernel at all (self.lag)."""
        if self.nu1 >= 1 and self.lag is not False:
            try:
                self._sweep(self.levels[0], norm=self.norm)
                self.lag = True
            except NotImplementedError:
                self.lag = False
        _zero(self.norm)

    def _host_scalar(self, t):
        """t (1-element device tensor) -> float via the pinned mailbox."""
        check(lib().amrb_store_host(C.c_void_p(t.data_ptr()), C.c_void_p(self.norm_host.data_ptr()), 1,
                                    stream_ptr()))
        torch.cuda.current_stream().synchronize()
        self._check_faults()
        return float(self.norm_host[0])

    def _check_faults(self):
        if self.dist and hasattr(self.transport, "check_faults"):
            self.transport.check_faults()

    # -- the device-side solve loop -------------------------------------------------
    _HIST = 4096  # capacity of the residual history (max_iter is capped to it)

    def _capture(self):
        """Warm up (lazy native tables, copy programs, scratch) on zeroed state,
        then capture one iteration into the body of a WHILE-node graph
        (csrc/graph.cu): a solve is one graph launch + one synchronisation."""
        for lv in self.levels:
            for f in lv.phi + [lv.rhs]:
                _zero(f)
                self._produced(f, f.ngrow)
        saved = [lv.cur for lv in self.levels]
        self._prime()
        self._body()
        self._body()  # both iterations start from the same state
        torch.cuda.synchronize()
        start = [lv.cur for lv in self.levels]
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        loop = C.c_void_p()
        with torch.cuda.stream(s):
            check(lib().amrb_loop_begin(stream_ptr(), C.byref(loop)))
            try:
                l0 = int(lib().amrb_launch_count())
                self._body()
                check(lib().amrb_loop_control(loop, C.c_void_p(self.norm.data_ptr()),
                                              C.c_void_p(self.r0_dev.data_ptr()),
                                              C.c_void_p(self.loop_dev.data_ptr()), self._HIST, stream_ptr()))
                self.launches_per_cycle = int(lib().amrb_launch_count()) - l0  # incl. the control kernel
            except BaseException:
                lib().amrb_loop_destroy(loop)
                raise
            check(lib().amrb_loop_end(loop))
        torch.cuda.current_stream().wait_stream(s)
        if [lv.cur for lv in self.levels] != start:
            lib().amrb_loop_destroy(loop)
            raise RuntimeError("captured iteration does not return the level buffers to their start state")
        self._loop = loop
        self._loop_cur = start
        self._loop_entry = saved  # buffer state set_phi / _prime start from
        for lv, c in zip(self.levels, saved):
            lv.cur = c

    def __del__(self):
        loop = getattr(self, "_loop", None)
        if loop is not None:
            try:
                lib().amrb_loop_destroy(loop)
            except Exception:
                pass

    # -- public API ----------------------------------------------------------------------
    def set_rhs(self, rhs):
        top = self.levels[0]
        parallel_copy(top.rhs, rhs, self.transport)
        self._produced(top.rhs, 0)
        self._need_ghosts(top, top.rhs, 1)

    def set_phi(self, phi):
        top = self.levels[0]
        if not self.all_periodic:
            # the finest level's 'external' ghosts (apply_domain_boundary), in
            # both ping-pong buffers: no kernel writes them afterwards
            for f in top.phi:
                self._domain_bc(top, f, 1, self.bc.external_value)
        parallel_copy(top.phi[top.cur], phi, self.transport)
        self._produced(top.phi[top.cur], 0)
        self._need_ghosts(top, top.phi[top.cur], 2)

    def get_phi(self, phi):
        top = self.levels[0]
        parallel_copy(phi, top.phi[self._solution_index()], self.transport)

    def solve(self, phi, rhs, rtol=1e-10, max_iter=200, wait=True):
        """Solve L(phi) = rhs to ||r||_inf <= rtol * ||rhs||_inf; phi is the
        initial guess and receives the solution.  Returns the final ||r||_inf;
        ``iterations``, ``history`` and ``r0`` are left on the solver.

        ``wait=False`` (graph solves): everything is queued on the current
        stream and the call returns None at once; ``finish()`` waits for the
        oldest queued solve and returns what solve() would have (so a caller
        can queue the next solve before reading this one: no idle device
        between solves).  At most two solves may be queued."""
        if len(self._queued) >= 2:
            raise RuntimeError("two solves already queued: call finish() first")
        max_iter = int(max_iter)
        if max_iter < 0 or max_iter > self._HIST:
            raise ValueError(f"max_iter must be in [0, {self._HIST}]")
        top = self.levels[0]
        if self.use_graph and self._loop is None:
            self._capture()
        if self._loop is not None:
            # the captured loop expects the primed sweep's output where the
            # capture left it: start every solve from the capture's entry
            # state (a previous solve leaves lv.cur at the loop's state)
            for lv, c in zip(self.levels, self._loop_entry):
                lv.cur = c
        self.set_rhs(rhs)
        self.set_phi(phi)
        device_reduce(top.rhs, "absmax", 0, out=self.r0_dev)
        self._allmax(self.r0_dev)
        self.history = []
        self.iterations = 0
        if max_iter == 0:
            self._drain()
            self.r0 = self._host_scalar(self.r0_dev)
            self.get_phi(phi)
            return self._done(self.r0, wait)
        self._prime()
        if self._loop is not None:
            for lv, c in zip(self.levels, self._loop_cur):
                lv.cur = c
            check(lib().amrb_loop_reset(C.c_void_p(self.loop_dev.data_ptr()), float(rtol), max_iter,
                                        C.c_void_p(self.r0_dev.data_ptr()), stream_ptr()))
            check(lib().amrb_loop_launch(self._loop, stream_ptr()))
            self.graph_replays += 1
            h = self.loop_host[self._host_slot]
            self._host_slot ^= 1
            check(lib().amrb_store_host(C.c_void_p(self.loop_dev.data_ptr()), C.c_void_p(h.data_ptr()),
                                        3 + max_iter, stream_ptr()))
            self.get_phi(phi)
            ev = torch.cuda.Event()
            ev.record()
            self._queued.append(("graph", h, ev))
            return self.finish() if wait else None
        else:
            self._drain()
            self.r0 = r0 = self._host_scalar(self.r0_dev)
            rn = r0
            while self.iterations < max_iter:
                self._body()
                self.iterations += 1
                rn = self._host_scalar(self.norm)
                _zero(self.norm)
                self.history.append(rn)
                if rn <= rtol * r0:
                    break
        self.get_phi(phi)
        return self._done(rn, wait)

    def _done(self, rn, wait):
        """A solve that finished synchronously: queue its result for finish()."""
        if wait:
            return rn
        self._queued.append(("done", (rn, self.r0, self.iterations, list(self.history)), None))
        return None

    def _drain(self):
        while self._queued:
            self.finish()

    def finish(self):
        """Wait for the oldest solve queued with solve(wait=False); sets r0,
        iterations and history from it and returns its final ||r||_inf."""
        if not self._queued:
            raise RuntimeError("no queued solve")
        kind, h, ev = self._queued.popleft()
        if kind == "done":
            rn, self.r0, self.iterations, self.history = h
            return rn
        ev.synchronize()
        self._check_faults()
        self.r0 = float(h[2])
        self.iterations = int(h.view(torch.int32)[3])
        self.history = [float(x) for x in h[3:3 + self.iterations].tolist()]
        return self.history[-1]


class _LocalView:
    """Transport facade for copies between a distributed FabArray and this
    rank's replica: the program keeps only records that are local to this rank."""

    def __init__(self, t):
        self.nranks = t.nranks
        self.rank = t.rank
        self.mode = "local"
        self.nccl_comm = None

    def account(self, *a):
        pass
