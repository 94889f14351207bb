"""Device-resident mesh data: Fab, FabArray and MultiFab.

Drop-in for the reference's containers (/root/reference/pkg/src/amrkit/
fabarray.py:28-131): same constructor ``FabArray(ba, dm, ncomp, ngrow,
dtype)``, same ``fab(i)`` accessor returning a Fab with ``box / gbox / ncomp
/ ngrow / data / valid() / slice() / setval()``, and ``data`` keeps the
reference's logical shape ``(ncomp, *grown extents)`` in C order (last axis
unit-stride).

What changes is where the bytes live.  A FabArray owns ONE torch CUDA
allocation per device; box b occupies a contiguous, 256-byte aligned block in
which every k-row (last axis) is padded so the first VALID cell of each row
starts on a 32-byte sector and the row pitch is a multiple of 4 doubles.
``fab(i).data`` is an ``as_strided`` view of that block with the logical
shape.  ``fabtab`` (int64, nboxes x 8) describes the layout to libamrb.

Ranks: in one process (the reference's simulated ranks, and the 1-GPU case)
every box is resident on the one device; under torch.distributed with one
process per GPU and ``dm.nranks == world_size`` only the boxes owned by this
rank are allocated (owner-computes).  ``replicated=True`` makes
every box resident on every rank (the agglomerated MLMG bottom levels).
"""

from __future__ import annotations

import numpy as np
import torch

from .boxes import Box, IntVect
from .layout import BoxArray, DistributionMapping

__all__ = ["Fab", "FabArray", "MultiFab", "ArrayView", "current_rank", "world_size"]

import itertools

_serials = itertools.count(1)
_ALIGN_ROW = 4  # doubles: 32-byte sectors
_ALIGN_BOX = 32  # doubles: 256 bytes


def world_size():
    import torch.distributed as dist

    if dist.is_available() and dist.is_initialized():
        return dist.get_world_size()
    return 1


def current_rank():
    import torch.distributed as dist

    if dist.is_available() and dist.is_initialized():
        return dist.get_rank()
    return 0


def _default_device():
    if torch.cuda.is_available():
        return torch.device("cuda", torch.cuda.current_device())
    return torch.device("cpu")


def _round(x, a):
    return (x + a - 1) // a * a


class Fab:
    """One box's data: a strided view into the owning FabArray's allocation."""

    __slots__ = ("box", "gbox", "ncomp", "ngrow", "data", "_owner", "_index_in_owner")

    def __init__(self, box, ncomp, ngrow, data, owner=None, index=-1):
        import weakref

        self.ngrow, self.ncomp = int(ngrow), int(ncomp)
        self.box, self.gbox, self.data = box, box.grow(int(ngrow)), data
        self._owner = weakref.ref(owner) if owner is not None else (lambda: None)
        self._index_in_owner = index

    def _index(self, region):
        if not self.gbox.contains_box(region):
            raise ValueError(f"{region!r} not within {self.gbox!r}")
        return tuple(slice(a - g, b - g + 1) for a, b, g in zip(region.lo, region.hi, self.gbox.lo))

    def slice(self, region, comp=None):
        """View of ``region`` (all components, or one)."""
        return self.data[(slice(None) if comp is None else comp,) + self._index(region)]

    def valid(self, comp=None):
        """View of the valid box."""
        return self.slice(self.box, comp)

    def array(self):
        """Global-index window onto this fab."""
        return ArrayView(self)

    def setval(self, value, comp=None, ghosts=True):
        """Valid (or grown) cells of one or all components = value, by the
        library's setval kernel on the owning FabArray (Fab.setval,
        fabarray.py:58-65)."""
        self._owner()._setval_boxes(value, comp, ghosts, box=self._index_in_owner)


class ArrayView:
    """Global-index window onto a Fab (fabarray.py:68-91): ``view[i, j, k, n]``
    -- the spatial indices are global cell indices, the last one the component."""

    __slots__ = ("data", "lo", "dim")

    def __init__(self, fab):
        self.data, self.lo, self.dim = fab.data, fab.gbox.lo, fab.box.dim

    def _local(self, key):
        if len(key) - 1 != self.dim:
            raise IndexError(f"expected {self.dim + 1} indices (spatial + component)")
        *cell, comp = key
        return (comp, *(c - o for c, o in zip(cell, self.lo)))

    def __getitem__(self, key):
        return self.data[self._local(key)]

    def __setitem__(self, key, value):
        self.data[self._local(key)] = value


class FabArray:
    """One Fab per box of ``ba``; boxes resident where ``dm`` puts them."""

    def __init__(self, ba, dm, ncomp=1, ngrow=0, dtype=np.float64, *, device=None, replicated=False, rank=None,
                 symmetric=False):
        if len(ba) != len(dm):
            raise ValueError("BoxArray and DistributionMapping lengths differ")
        if np.dtype(dtype) != np.float64:
            raise ValueError("device FabArrays hold float64 (the reference's MultiFab type)")
        self.ba = ba
        self.dm = dm
        self.ncomp = int(ncomp)
        self.ngrow = int(ngrow)
        self.dtype = np.dtype(np.float64)
        self.device = torch.device(device) if device is not None else _default_device()
        self.replicated = bool(replicated)
        ws = world_size()
        self.distributed = (not replicated) and ws > 1 and dm.nranks == ws
        self.rank = current_rank() if rank is None else int(rank)
        if self.distributed:
            self.resident = np.array([r == self.rank for r in dm.owner], dtype=bool)
        else:
            self.resident = np.ones(len(ba), dtype=bool)
        self._layout()
        # symmetric: one process per GPU, storage in torch symmetric memory so
        # every peer can read this rank's boxes over NVLink (p2p ghost fills)
        self.symmetric = bool(symmetric) and self.distributed
        self.peer_ptrs = None
        if self.symmetric:
            import torch.distributed as dist
            import torch.distributed._symmetric_memory as symm_mem

            n = torch.tensor([self._nelems], dtype=torch.int64, device=self.device)
            dist.all_reduce(n, op=dist.ReduceOp.MAX)
            self.storage = symm_mem.empty(int(n.item()), dtype=torch.float64, device=self.device)
            self.storage.zero_()
            self._symm = symm_mem.rendezvous(self.storage, dist.group.WORLD.group_name)
            self.peer_ptrs = np.array(self._symm.buffer_ptrs, dtype=np.uint64)
        else:
            self.storage = torch.zeros(self._nelems, dtype=torch.float64, device=self.device)
        self.fabs = {}
        for i in range(len(ba)):
            if self.resident[i]:
                self.fabs[i] = Fab(ba[i], self.ncomp, self.ngrow, self._view(i), self, i)
        self._progs = {}
        self._native = {}
        self.serial = next(_serials)

    # -- layout ---------------------------------------------------------------
    def global_fabtab(self):
        """Every box's layout inside its OWNER's allocation (p2p copy sources)."""
        if getattr(self, "_gtab", None) is None:
            keep = self.resident
            tab = np.zeros_like(self.fabtab)
            for r in range(self.dm.nranks):
                self.resident = np.array([o == r for o in self.dm.owner], dtype=bool)
                saved = (self.fabtab, self._ext3, self._nelems)
                self._layout()
                rows = self.resident
                tab[rows] = self.fabtab[rows]
                self.fabtab, self._ext3, self._nelems = saved
            self.resident = keep
            self._gtab = tab
        return self._gtab

    def _layout(self):
        dim = self.ba.dim
        pad = 3 - dim
        g = self.ngrow
        n = len(self.ba)
        tab = np.zeros((n, 8), dtype=np.int64)
        ext3 = np.ones((n, 3), dtype=np.int64)
        front = (_ALIGN_ROW - g % _ALIGN_ROW) % _ALIGN_ROW
        off = 0
        for i, b in enumerate(self.ba):
            e = [1, 1, 1]
            glo = [0, 0, 0]
            for d in range(dim):
                e[pad + d] = b.hi[d] - b.lo[d] + 1 + 2 * g
                glo[pad + d] = b.lo[d] - g
            ext3[i] = e
            pitch = _round(front + e[2] + 2, _ALIGN_ROW)
            s1 = pitch
            s0 = e[1] * s1
            cs = e[0] * s0
            if self.resident[i]:
                tab[i] = (off + front, cs, s0, s1, glo[0], glo[1], glo[2], 1)
                off += _round(self.ncomp * cs, _ALIGN_BOX)
            else:
                tab[i, 4:7] = glo
        self.fabtab = tab
        self._ext3 = ext3
        self._nelems = max(off + _ALIGN_BOX, _ALIGN_BOX)

    def _view(self, i):
        t = self.fabtab[i]
        dim = self.ba.dim
        pad = 3 - dim
        size = (self.ncomp,) + tuple(int(x) for x in self._ext3[i][pad:])
        all_strides = (int(t[1]), int(t[2]), int(t[3]), 1)
        stride = (all_strides[0],) + all_strides[1 + pad :]
        return torch.as_strided(self.storage, size, stride, int(t[0]))

    @property
    def dim(self):
        return self.ba.dim

    def fab(self, i):
        try:
            return self.fabs[i]
        except KeyError:
            raise KeyError(f"box {i} is not resident on rank {self.rank}") from None

    def local_indices(self, rank=None):
        if rank is None:
            return [i for i in range(len(self.ba)) if self.resident[i]]
        return self.dm.owned_indices(rank)

    def setval(self, value, comp=None, ghosts=True):
        """Every resident fab (fabarray.py:119-122), by library kernels: the
        whole allocation (padding included) in one fill when ghosts and all
        components are set, else the setval kernel over the boxes."""
        self.require_cuda("setval")
        from ._native import check, lib
        from .device import stream_ptr

        if ghosts and comp is None:
            import ctypes as C

            check(lib().amrb_fill(C.c_void_p(self.storage.data_ptr()), self.storage.numel(), float(value),
                                  stream_ptr()))
            return self
        return self._setval_boxes(value, comp, ghosts)

    def _setval_boxes(self, value, comp=None, ghosts=True, box=-1):
        import ctypes as C

        from ._native import check, lib
        from .device import field_of, level_of, stream_ptr

        self.require_cuda("setval")
        c0, c1 = (0, self.ncomp) if comp is None else (int(comp), int(comp) + 1)
        if not 0 <= c0 < c1 <= self.ncomp:
            raise ValueError("component out of range")
        mode = 2 if ghosts == 2 else (1 if ghosts else 0)
        check(lib().amrb_setval(level_of(self).handle, field_of(self).handle, C.c_void_p(self.storage.data_ptr()),
                                int(box), c0, c1, mode, float(value), stream_ptr()))
        return self

    def copy_shape(self, ncomp=None, ngrow=None):
        """A new zeroed FabArray on the same layout and device."""
        nc = self.ncomp if ncomp is None else ncomp
        ng = self.ngrow if ngrow is None else ngrow
        return type(self)(self.ba, self.dm, nc, ng, self.dtype, device=self.device, replicated=self.replicated,
                          rank=self.rank)

    def owners(self):
        """Owner rank per box as seen by copy programs.

        A replicated FabArray is resident everywhere, so under one process per
        GPU every box counts as owned by this rank (copies from/to it are local).
        """
        if self.replicated and world_size() > 1:
            return np.full(len(self.ba), self.rank, dtype=np.int32)
        return np.asarray(self.dm.owner, dtype=np.int32)

    # -- host <-> device helpers ----------------------------------------------
    # -- bulk host <-> device (one contiguous copy + one launch each way) -------
    def image_size(self):
        """Elements of the host image: every RESIDENT box's valid region,
        comp-major C order, boxes back to back in index order (the plotfile
        data.bin record layout restricted to this rank's boxes)."""
        return self.ncomp * sum(self.ba[i].num_cells() for i in range(len(self.ba)) if self.resident[i])

    def from_host_image(self, image, stream=None):
        """Valid cells of resident boxes <- a host image (pinned float64 tensor of
        image_size() elements, see image_size): one async host->device copy
        into a cached device staging buffer and one scatter launch, both on
        `stream` (default: current).  The caller keeps `image` alive until the
        copy has run."""
        from .plotfile import _packer

        st = stream if stream is not None else torch.cuda.current_stream(self.device)
        stage = self._native.get("img_in")
        if stage is None:
            stage = torch.empty(max(self.image_size(), 1), dtype=torch.float64, device=self.device)
            self._native["img_in"] = stage
        with torch.cuda.stream(st):
            stage[: image.numel()].copy_(image, non_blocking=True)
            _packer(self, False, compact=True).run(stage.data_ptr(), self.storage.data_ptr())
        return self

    def to_host_image(self, image, stream=None):
        """host image (pinned float64, image_size() elements) <- valid cells of
        resident boxes: one gather launch + one async device->host copy on
        `stream`; synchronize before reading `image`."""
        from .plotfile import _packer

        st = stream if stream is not None else torch.cuda.current_stream(self.device)
        stage = self._native.get("img_out")
        if stage is None:
            stage = torch.empty(max(self.image_size(), 1), dtype=torch.float64, device=self.device)
            self._native["img_out"] = stage
        with torch.cuda.stream(st):
            _packer(self, True, compact=True).run(self.storage.data_ptr(), stage.data_ptr())
            image.copy_(stage[: image.numel()], non_blocking=True)
        return image

    def load_valid_from(self, domain, global_arr):
        """Load every resident fab's valid region from one dense array over
        domain: the host gathers the boxes into the host-image layout
        (image_size), then one host->device copy and one scatter launch
        (from_host_image)."""
        g = np.asarray(global_arr, dtype=np.float64)
        if g.ndim == self.dim:
            g = g[None]
        if g.shape[0] != self.ncomp:
            raise ValueError("component count differs")
        image = torch.empty(max(self.image_size(), 1), dtype=torch.float64).pin_memory()
        flat = image.numpy()
        o = 0
        for i in range(len(self.ba)):
            if not self.resident[i]:
                continue
            b = self.ba[i]
            sel = tuple(slice(b.lo[d] - domain.lo[d], b.hi[d] - domain.lo[d] + 1) for d in range(self.dim))
            blk = g[(slice(None),) + sel]
            flat[o:o + blk.size] = blk.reshape(-1)
            o += blk.size
        self.from_host_image(image[: self.image_size()])
        torch.cuda.current_stream(self.device).synchronize()  # the pinned image is released on return
        return self

    def to_global(self, domain, comp=0, default=0.0):
        """Dense numpy array over domain from resident valid data."""
        from .comm import gather_global

        return gather_global(self, domain, comp, default)

    def require_cuda(self, what):
        if self.device.type != "cuda":
            raise RuntimeError(f"{what}: FabArray storage is on {self.device}; the hot path runs on CUDA only")


class MultiFab(FabArray):
    """float64 FabArray (AMReX's MultiFab)."""
