"""Ghost exchange, inter-layout copy, boundary folding and reductions.

Drop-in for the reference's FabArray communication API
(/root/reference/pkg/src/amrkit/fabarray.py:364-455) and its Transport
(transport.py:20-58):

    fill_boundary(fa, transport, domain, periodic=None)      fabarray.py:364
    parallel_copy(dst, src, transport, domain=None, periodic=None)  :377
    sum_boundary(fa, transport, domain, periodic=None)       :391
    reduce(fa, kind, comp, transport)                        :409
    gather_global(fa, region, comp=0, default=0.0)           :443

Execution is a libamrb copy program (csrc/comm.cu) running on the current
torch CUDA stream: one kernel launch for all local records, pack/unpack
kernels around one message per ordered rank pair for remote ones.  A
``Transport(nranks)`` simulates ranks inside one process exactly like the
reference (all boxes on one GPU, messages counted); ``Transport.distributed()``
is the real thing -- one process per GPU, messages are NCCL send/recv.
"""

from __future__ import annotations

import ctypes as C
from collections import defaultdict, deque

import numpy as np
import torch

from . import counters
from ._native import AMRB_ENOTSUP, check, i32p, i64p, lib, ptr
from .boxes import box_diff
from .device import field_of, level_of, stream_ptr
from .plans import (
    build_plan_copy,
    build_plan_copy_grown,
    build_plan_fill_boundary,
    build_plan_sum_boundary,
    normalize_periodic,
)

__all__ = [
    "Transport",
    "TransportError",
    "fill_boundary",
    "parallel_copy",
    "sum_boundary",
    "reduce",
    "gather_global",
    "copy_into",
]


class TransportError(RuntimeError):
    """A message between two ranks failed (transport.py:20-24): ``src``,
    ``dst`` and the reason in the message."""

    def __init__(self, src, dst, why):
        self.src, self.dst = src, dst
        super().__init__(f"transport failure {src} -> {dst}: {why}")


class Transport:
    """Message layer between ranks.

    ``Transport(nranks)``: the reference's simulated ranks (transport.py:27-58)
    -- every rank lives in this process; device messages are segments of one
    staging buffer on the GPU; host messages use FIFO mailboxes.
    ``Transport.distributed()``: one process per GPU under torch.distributed;
    device messages travel by NCCL send/recv over NVLink.
    """

    def __init__(self, nranks):
        if int(nranks) < 1:
            raise ValueError("nranks must be >= 1")
        self.nranks, self.rank, self.mode = int(nranks), 0, "sim"
        self.nccl_comm, self.p2p = None, False
        self._queues = defaultdict(deque)  # (src, dst) -> FIFO of (tag, payload)

    @classmethod
    def distributed(cls):
        import torch.distributed as dist

        if not (dist.is_available() and dist.is_initialized()):
            raise ValueError("Transport.distributed() needs torch.distributed to be initialised")
        t = cls(dist.get_world_size())
        t.rank = dist.get_rank()
        t.mode = "nccl"
        uid = (C.c_uint8 * 128)()
        if t.rank == 0:
            check(lib().amrb_nccl_unique_id(uid))
        obj = [bytes(uid)]
        dist.broadcast_object_list(obj, src=0)
        uid = (C.c_uint8 * 128).from_buffer_copy(obj[0])
        comm = C.c_void_p()
        check(lib().amrb_nccl_comm_create(uid, t.nranks, t.rank, C.byref(comm)), src=t.rank, dst=-1)
        t.nccl_comm = comm
        t._setup_p2p()
        return t

    def _setup_p2p(self):
        """Signal pads + device epoch for the NVLink barrier of p2p fills."""
        self.p2p = False
        if self.nranks > 8:
            return
        try:
            import torch.distributed as dist
            import torch.distributed._symmetric_memory as symm_mem

            dev = torch.device("cuda", torch.cuda.current_device())
            self._bar_buf = symm_mem.empty(64, dtype=torch.int32, device=dev)
            self._bar = symm_mem.rendezvous(self._bar_buf, dist.group.WORLD.group_name)
            self._pads = np.array(self._bar.signal_pad_ptrs, dtype=np.uint64)
            # peer_allmax: 2 epoch-tagged uint64 words per rank, zero before first use
            self._slots_buf = symm_mem.empty(16, dtype=torch.float64, device=dev)
            self._slots_buf.zero_()
            self._slots = symm_mem.rendezvous(self._slots_buf, dist.group.WORLD.group_name)
            self._slot_ptrs = np.array(self._slots.buffer_ptrs, dtype=np.uint64)
            self._epoch = torch.zeros(2, dtype=torch.int32, device=dev)  # epoch, CTA ticket
            # pads start at zero; make sure every rank sees that before the first barrier
            self._bar.barrier()
            torch.cuda.synchronize()
            ok = True
        except Exception:  # no symmetric memory on this system: NCCL send/recv only
            ok = False
        # device-side peer waits report a missing peer here (amrb_set_fault_mailbox)
        self._faults = torch.zeros(4, dtype=torch.int64).pin_memory()
        check(lib().amrb_set_fault_mailbox(C.c_void_p(self._faults.data_ptr())))
        # every rank must take the same path: enable p2p only if it worked everywhere
        import torch.distributed as dist

        flag = torch.tensor([1 if ok else 0], dtype=torch.int32, device=torch.device("cuda", torch.cuda.current_device()))
        dist.all_reduce(flag, op=dist.ReduceOp.MIN)
        self.p2p = bool(flag.item())

    def peer_allmax(self, t):
        """t (1-element float64 CUDA tensor) <- max over ranks, over NVLink."""
        check(
            lib().amrb_peer_allmax(
                self._pads.ctypes.data_as(C.POINTER(C.c_uint64)),
                self._slot_ptrs.ctypes.data_as(C.POINTER(C.c_uint64)),
                self.rank,
                self.nranks,
                C.c_void_p(self._epoch.data_ptr()),
                C.c_void_p(t.data_ptr()),
                stream_ptr(),
            ),
            src=self.rank,
        )

    def check_faults(self):
        """Raise TransportError(rank, peer) if a device-side wait for a peer
        timed out (library option "peer_timeout_ms").  Call after synchronising
        the stream the waits ran on."""
        f = getattr(self, "_faults", None)
        if f is None or int(f[0]) == 0:
            return
        code, me, peer, epoch = (int(x) for x in f.tolist())
        from ._native import get_option

        raise TransportError(peer, me, f"peer {peer} did not reach device epoch {epoch} within "
                                       f"{get_option('peer_timeout_ms')} ms (NVLink signal wait, code {code})")

    def peer_barrier(self):
        check(
            lib().amrb_peer_barrier(
                self._pads.ctypes.data_as(C.POINTER(C.c_uint64)),
                self.rank,
                self.nranks,
                C.c_void_p(self._epoch.data_ptr()),
                stream_ptr(),
            ),
            src=self.rank,
        )

    def close(self):
        """Destroy the NCCL communicator.  Call only after every CUDA graph that
        captured operations on it has been released (ncclCommDestroy otherwise
        waits for them); at process exit it can simply be left to the OS."""
        if self.nccl_comm is not None and self.nccl_comm.value:
            check(lib().amrb_nccl_comm_destroy(self.nccl_comm))
            self.nccl_comm = None

    # -- host message API (reference-compatible) -------------------------------
    def send(self, src, dst, tag, payload):
        if not (0 <= src < self.nranks and 0 <= dst < self.nranks):
            raise TransportError(src, dst, "rank out of range")
        self._queues[(src, dst)].append((tag, payload))
        self.account(src, dst, int(getattr(payload, "nbytes", len(payload))))

    def drain(self, dst):
        """Every message queued for ``dst``, by source rank, FIFO per source."""
        got = []
        for src in range(self.nranks):
            q = self._queues.pop((src, dst), None)
            got.extend((src, tag, payload) for tag, payload in (q or ()))
        return got

    def pending(self):
        return sum(map(len, self._queues.values()))

    def account(self, src, dst, nbytes):
        counters.incr("transport_messages")
        counters.incr("transport_bytes", int(nbytes))


class _Program:
    """A plan bound to (src storage, dst storage, transport mode)."""

    def __init__(self, plan, src_fa, dst_fa, transport, op, p2p=False):
        self.plan = plan  # keep the native plan alive
        self.p2p = p2p
        sim = transport.mode == "sim"
        mode = 3 if p2p else {"nccl": 0, "sim": 1, "local": 2}[transport.mode]
        ncomp = src_fa.ncomp
        st, stp = i64p(src_fa.global_fabtab() if p2p else src_fa.fabtab)
        dt, dtp = i64p(dst_fa.fabtab)
        so, sop = i32p(src_fa.owners())
        do, dop = i32p(dst_fa.owners())
        h = C.c_void_p()
        check(
            lib().amrb_prog_create(
                plan.handle,
                ncomp,
                stp,
                len(src_fa.ba),
                sop,
                dtp,
                len(dst_fa.ba),
                dop,
                transport.nranks,
                transport.rank,
                mode,
                op,
                C.byref(h),
            )
        )
        self.handle = h
        send = C.c_int64()
        recv = C.c_int64()
        npairs = C.c_int64()
        nlocal = C.c_int64()
        check(lib().amrb_prog_info(h, C.byref(send), C.byref(recv), C.byref(npairs), C.byref(nlocal)))
        pairs = np.zeros((npairs.value, 4), dtype=np.int64)
        if npairs.value:
            check(lib().amrb_prog_pairs(h, pairs.ctypes.data_as(C.POINTER(C.c_int64))))
        self.pairs = pairs
        dev = dst_fa.device
        self.sendbuf = torch.empty(max(send.value, 1), dtype=torch.float64, device=dev) if send.value else None
        self.recvbuf = (
            torch.empty(max(recv.value, 1), dtype=torch.float64, device=dev) if (recv.value and not sim) else None
        )

    def __del__(self):
        h = getattr(self, "handle", None)
        if h is not None and h.value:
            try:
                lib().amrb_prog_destroy(h)
            except Exception:
                pass

    def run(self, src_fa, dst_fa, transport, post_barrier=True):
        if self.p2p:
            # pull model: peers' boxes are final once everyone reached this point;
            # the barrier is fused into the copy launch (k_copy, SyncArgs)
            check(
                lib().amrb_prog_run_p2p_sync(
                    self.handle,
                    C.c_void_p(src_fa.storage.data_ptr()),
                    C.c_void_p(dst_fa.storage.data_ptr()),
                    src_fa.peer_ptrs.ctypes.data_as(C.POINTER(C.c_uint64)),
                    transport.nranks,
                    transport._pads.ctypes.data_as(C.POINTER(C.c_uint64)),
                    transport.rank,
                    C.c_void_p(transport._epoch.data_ptr()),
                    stream_ptr(),
                ),
                src=transport.rank,
            )
            if post_barrier:  # nobody may overwrite what a peer is still reading
                transport.peer_barrier()
            return
        comm = transport.nccl_comm if transport.mode == "nccl" else None
        if transport.mode == "local":
            comm = None
        check(
            lib().amrb_prog_run(
                self.handle,
                C.c_void_p(src_fa.storage.data_ptr()),
                C.c_void_p(dst_fa.storage.data_ptr()),
                C.c_void_p(ptr(self.sendbuf)),
                C.c_void_p(ptr(self.recvbuf)),
                comm,
                stream_ptr(),
            ),
            src=transport.rank,
        )
        for s, d, _off, cnt in self.pairs.tolist():
            transport.account(s, d, 8 * cnt)


def _execute(plan, src_fa, dst_fa, transport, op, post_barrier=True):
    nranks = transport.nranks
    if src_fa.dm.nranks != nranks or dst_fa.dm.nranks != nranks:
        raise ValueError("transport rank count differs from the distribution maps")
    src_fa.require_cuda("copy")
    dst_fa.require_cuda("copy")
    p2p = transport.mode == "nccl" and transport.p2p and getattr(src_fa, "symmetric", False)
    if op == 2 and not p2p:
        raise ValueError("a local-sources fill needs the p2p transport (symmetric storage)")
    key = (id(plan), src_fa.serial, op, transport.mode, nranks, p2p)
    prog = dst_fa._progs.get(key)
    if prog is None:
        prog = _Program(plan, src_fa, dst_fa, transport, op, p2p=p2p)
        dst_fa._progs[key] = prog
    prog.run(src_fa, dst_fa, transport, post_barrier=post_barrier)


def fill_boundary(fa, transport, domain, periodic=None, ngrow=None, _post_barrier=True, _local_sources=False):
    """Fill every in-domain (or periodic-image) ghost cell from the valid cell it
    shadows; out-of-domain non-periodic ghosts are untouched (fabarray.py:364).

    ``ngrow`` (<= fa.ngrow) limits the exchange to the first ``ngrow`` ghost
    layers (AMReX FillBoundary(nghost)); default is all of them.
    ``_local_sources`` (p2p transport only; the MLMG's remote ghost push) copies
    only the ghost cells whose source box lives on this GPU -- peers already
    stored the rest -- and is the device barrier that makes those stores
    visible before the next kernel.
    """
    ng = fa.ngrow if ngrow is None else int(ngrow)
    if ng > fa.ngrow:
        raise ValueError("fill width exceeds the FabArray's ghost width")
    if ng == 0:
        return
    if _single_periodic_box(fa, transport, domain, periodic, _local_sources):
        # one box that is the whole periodic domain: every ghost is a wrapped
        # copy of the box itself -- one record-free launch (amrb_fill_wrap)
        fa.require_cuda("fill_boundary")
        rc = lib().amrb_fill_wrap(level_of(fa).handle, field_of(fa).handle, C.c_void_p(fa.storage.data_ptr()),
                                  fa.ncomp, ng, stream_ptr())
        if rc == 0:
            return
        if rc != AMRB_ENOTSUP:
            check(rc)
    plan = build_plan_fill_boundary(fa.ba, ng, domain, periodic)
    _execute(plan, fa, fa, transport, 2 if _local_sources else 0, post_barrier=_post_barrier)


def _single_periodic_box(fa, transport, domain, periodic, local_sources):
    # one process, or a replicated FabArray (every rank holds the whole box:
    # the fill involves no peer)
    if local_sources or fa.dim != 3 or len(fa.ba) != 1 or domain is None:
        return False
    if transport.nranks != 1 and not getattr(fa, "replicated", False):
        return False
    if not all(normalize_periodic(periodic, fa.dim)):
        return False
    b = fa.ba[0]
    return tuple(b.lo) == tuple(domain.lo) and tuple(b.hi) == tuple(domain.hi) and bool(fa.resident[0])


def parallel_copy(dst_fa, src_fa, transport, domain=None, periodic=None):
    """Copy src valid data onto dst valid cells wherever layouts overlap (:377)."""
    if dst_fa.ncomp != src_fa.ncomp:
        raise ValueError(f"component count mismatch: dst {dst_fa.ncomp} vs src {src_fa.ncomp}")
    plan = build_plan_copy(dst_fa.ba, src_fa.ba, domain, periodic)
    _execute(plan, src_fa, dst_fa, transport, 0)


def copy_into(dst_fa, src_fa, transport, include_dst_ghosts=False, domain=None, periodic=None):
    """parallel_copy that may also write dst ghost cells (coarse_fine.py:188-198)."""
    if dst_fa.ncomp != src_fa.ncomp:
        raise ValueError("component count mismatch")
    ng = dst_fa.ngrow if include_dst_ghosts else 0
    plan = build_plan_copy_grown(dst_fa.ba, src_fa.ba, ng, domain, periodic)
    _execute(plan, src_fa, dst_fa, transport, 0)


def sum_boundary(fa, transport, domain, periodic=None):
    """Fold every ghost copy back onto its valid cell, in plan order, then zero
    the ghosts (fabarray.py:391-406)."""
    if fa.ngrow == 0:
        return
    plan = build_plan_sum_boundary(fa.ba, fa.ngrow, domain, periodic)
    _execute(plan, fa, fa, transport, 1)
    fa._setval_boxes(0.0, None, ghosts=2)  # ghost cells only (setval kernel)


_KINDS = {"sum": 0, "min": 1, "max": 2, "absmax": 3}


def device_reduce(fa, kind, comp=0, out=None):
    """Reduce over resident valid cells on this device into a 1-element tensor
    (no host sync).  kind in sum/min/max/absmax."""
    fa.require_cuda("reduce")
    if out is None:
        out = torch.empty(1, dtype=torch.float64, device=fa.device)
    lv = level_of(fa)
    f = field_of(fa)
    check(
        lib().amrb_reduce(
            lv.handle, f.handle, C.c_void_p(fa.storage.data_ptr()), comp, _KINDS[kind], C.c_void_p(out.data_ptr()),
            stream_ptr(),
        )
    )
    return out


def reduce(fa, kind, comp, transport):
    """Reduce one component over valid cells and combine across ranks (:409)."""
    if kind not in ("sum", "min", "max"):
        raise ValueError(f"unknown reduction {kind!r}")
    if not 0 <= comp < fa.ncomp:
        raise ValueError("component out of range")
    if transport.mode == "nccl" and (not fa.distributed or fa.dm.nranks != transport.nranks):
        # a replicated (or undistributed) FabArray holds every box on every rank:
        # summing the per-rank partials would count each box nranks times
        raise ValueError("reduce over NCCL needs a FabArray distributed over the transport's ranks")
    out = device_reduce(fa, kind, comp)
    if transport.mode == "nccl":
        check(
            lib().amrb_nccl_allreduce(
                C.c_void_p(out.data_ptr()), 1, _KINDS[kind], transport.nccl_comm, stream_ptr()
            ),
            src=transport.rank,
        )
        if transport.rank != 0:
            transport.account(transport.rank, 0, 8)
    else:
        # partials of ranks 1..R-1 travel to rank 0 in the reference
        for r in range(1, transport.nranks):
            transport.account(r, 0, 8)
    return float(out.item())


def gather_global(fa, region, comp=0, default=0.0):
    """Dense numpy array over region from resident valid data (diagnostics)."""
    out = np.full(tuple(region.extents()), default, dtype=np.float64)
    for i, f in fa.fabs.items():
        ov = fa.ba[i].intersect(region)
        if ov.is_empty():
            continue
        idx = tuple(slice(ov.lo[d] - region.lo[d], ov.hi[d] - region.lo[d] + 1) for d in range(fa.dim))
        out[idx] = f.slice(ov, comp).cpu().numpy()
    return out
