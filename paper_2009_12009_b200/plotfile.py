"""Plotfile / checkpoint I/O for device MultiFabs.

Drop-in for the mesh half of ``amrkit.plotfile``
(/root/reference/pkg/src/amrkit/plotfile.py:1-524, format in
/root/reference/pkg/FORMAT.md:17-84,128-160): same API (``OutputMode``,
``WriteHandle``, ``PlotfileHeader``, ``write_plotfile``, ``read_plotfile``,
``write_checkpoint``, ``read_checkpoint``), same counters (``io_waves``,
``io_peak_writers``, ``io_bytes_written``) and byte-identical files.

Device path:

* pack: ONE copy-program launch (csrc/comm.cu ``k_copy``) gathers every
  resident box's valid region into a device staging buffer laid out exactly as
  ``data.bin`` -- per box a comp-major, C-order ``<f8`` record at the offset
  the header prints (``_record_layout``, plotfile.py:160-169).  It runs on the
  caller's stream, so the snapshot is ordered before any later mutation;
* one device->host copy of the staging buffer into pinned memory (its own
  stream), then positioned writes (``os.pwrite``) per rank in waves of
  ``nwriters`` (plotfile.py:195-241) -- each record is written straight from
  the pinned image, no per-box host copies;
* ``OutputMode.asynchronous()``: the pack is enqueued at submit time, the
  copy-out and the file writes run on the single background writer thread
  (queue of one, plotfile.py:86-115) while the GPU keeps computing.

With one process per GPU every rank packs and writes its own boxes; rank 0
writes the Header and sizes the file first.
"""

from __future__ import annotations

import ctypes as C
import os
import queue
import threading

import numpy as np
import torch

from . import counters
from ._native import check, i32p, i64p, lib
from .boxes import Box, IntVect
from .device import stream_ptr
from .geometry import Geometry
from .layout import BoxArray, DistributionMapping
from .multifab import FabArray, world_size
from .plans import build_plan_copy

__all__ = [
    "PLOTFILE_TAG",
    "CHECKPOINT_TAG",
    "OutputMode",
    "WriteHandle",
    "PlotfileHeader",
    "write_plotfile",
    "read_plotfile",
    "write_checkpoint",
    "read_checkpoint",
]

PLOTFILE_TAG = "amrkit-plotfile-1"
CHECKPOINT_TAG = "amrkit-checkpoint-1"


class OutputMode:
    """``static(nwriters)`` writes now in waves; ``asynchronous()`` snapshots
    and returns (plotfile.py:43-64)."""

    __slots__ = ("kind", "nwriters")

    def __init__(self, kind, nwriters=1):
        if kind not in ("static", "async"):
            raise ValueError("mode kind must be 'static' or 'async'")
        if int(nwriters) < 1:
            raise ValueError("nwriters must be >= 1")
        self.kind = kind
        self.nwriters = int(nwriters)

    @staticmethod
    def static(nwriters=1):
        return OutputMode("static", nwriters)

    @staticmethod
    def asynchronous():
        return OutputMode("async")

    def __repr__(self):
        return f"OutputMode({self.kind}, nwriters={self.nwriters})"


class WriteHandle:
    """Completion of one write; ``wait()`` re-raises the writer's error."""

    def __init__(self):
        self._event = threading.Event()
        self._error = None

    def _finish(self, error=None):
        self._error = error
        self._event.set()

    @property
    def done(self):
        return self._event.is_set()

    def wait(self, timeout=None):
        if not self._event.wait(timeout):
            raise TimeoutError("write did not complete in time")
        if self._error is not None:
            raise self._error


class _Writer:
    """One background writer thread, at most one snapshot pending."""

    def __init__(self):
        self._queue = queue.Queue(maxsize=1)
        self._thread = None
        self._lock = threading.Lock()

    def _run(self):
        while True:
            job, handle = self._queue.get()
            try:
                job()
                handle._finish()
            except BaseException as exc:  # surfaced by handle.wait()
                handle._finish(exc)

    def submit(self, job):
        with self._lock:
            if self._thread is None or not self._thread.is_alive():
                self._thread = threading.Thread(target=self._run, daemon=True, name="amrb-plotfile-writer")
                self._thread.start()
        handle = WriteHandle()
        self._queue.put((job, handle))  # blocks while a snapshot is pending
        return handle


_writer = _Writer()


class PlotfileHeader:
    """Time, component names and one Geometry per level (plotfile.py:123-138)."""

    def __init__(self, time, names, geoms):
        self.version = PLOTFILE_TAG
        self.time = float(time)
        self.names = list(names)
        if any(" " in n for n in self.names):
            raise ValueError("component names may not contain spaces")
        self.geoms = list(geoms)

    @property
    def nlevels(self):
        return len(self.geoms)


def _floats(vals):
    return " ".join(repr(float(v)) for v in vals)


def _ints(vals):
    return " ".join(str(int(v)) for v in vals)


def _box_text(b):
    return _ints(tuple(b.lo) + tuple(b.hi))


def _record_layout(ba, ncomp):
    """Byte offset and size of every box record, and the file size."""
    sizes = [8 * ncomp * ba[i].num_cells() for i in range(len(ba))]
    offsets = np.concatenate(([0], np.cumsum(sizes)[:-1])).astype(np.int64) if sizes else np.zeros(0, np.int64)
    return [int(x) for x in offsets], sizes, int(sum(sizes))


def _header_text(header, meshes):
    g0 = header.geoms[0]
    out = [
        PLOTFILE_TAG,
        "endian little",
        "real float64",
        f"time {header.time!r}",
        f"dim {g0.dim}",
        f"nlevels {header.nlevels}",
        f"components {len(header.names)} " + " ".join(header.names),
        "prob_lo " + _floats(g0.prob_lo),
        "prob_hi " + _floats(g0.prob_hi),
        "periodic " + _ints(g0.periodic),
    ]
    for lev, mesh in enumerate(meshes):
        geom = header.geoms[lev]
        offs, sizes, _ = _record_layout(mesh.ba, mesh.ncomp)
        out += [f"level {lev}", "domain " + _box_text(geom.domain), "cell_size " + _floats(geom.cell_size),
                f"nboxes {len(mesh.ba)}"]
        out += [f"box {_box_text(mesh.ba[i])} {offs[i]} {sizes[i]}" for i in range(len(mesh.ba))]
    return "\n".join(out) + "\n"


# ---------------------------------------------------------------------------
# device staging: the data.bin image of one level
# ---------------------------------------------------------------------------


def _staging_fabtab(ba, offsets, resident):
    """Fab table describing the record layout: box i = comp-major C-order block
    at element offset offsets[i] / 8, no ghosts (3-D padded like multifab)."""
    dim = ba.dim
    pad = 3 - dim
    tab = np.zeros((len(ba), 8), dtype=np.int64)
    for i, b in enumerate(ba):
        e = [1, 1, 1]
        lo = [0, 0, 0]
        for d in range(dim):
            e[pad + d] = b.hi[d] - b.lo[d] + 1
            lo[pad + d] = b.lo[d]
        tab[i] = (offsets[i] // 8, e[0] * e[1] * e[2], e[1] * e[2], e[2], lo[0], lo[1], lo[2], 1 if resident[i] else 0)
    return tab


class _Packer:
    """Copy program between a FabArray and its data.bin staging image (either
    direction), cached on the FabArray.  compact=True: records of this rank's
    resident boxes only, back to back (FabArray host images)."""

    def __init__(self, fa, to_staging, compact=False):
        self.offsets, self.sizes, self.total = _record_layout(fa.ba, fa.ncomp)
        if compact:
            at = 0
            for i in range(len(fa.ba)):
                n = self.sizes[i] if fa.resident[i] else 0
                self.offsets[i], self.sizes[i] = at, n
                at += n
            self.total = at
        owners = fa.owners()
        nranks = fa.dm.nranks if world_size() > 1 else 1
        rank = fa.rank if world_size() > 1 else 0
        if nranks == 1:
            owners = np.zeros(len(fa.ba), dtype=np.int32)
        self.mine = [bool(fa.resident[i]) for i in range(len(fa.ba))]
        stab = _staging_fabtab(fa.ba, self.offsets, fa.resident)
        plan = build_plan_copy(fa.ba, fa.ba)
        self.plan = plan
        ft, ftp = i64p(fa.fabtab)
        st, stp = i64p(stab)
        ow, owp = i32p(np.ascontiguousarray(owners, dtype=np.int32))
        src, dst = (ftp, stp) if to_staging else (stp, ftp)
        h = C.c_void_p()
        check(lib().amrb_prog_create(plan.handle, fa.ncomp, src, len(fa.ba), owp, dst, len(fa.ba), owp, nranks, rank,
                                     2, 0, C.byref(h)))
        self.handle = h
        self._keep = (ft, st, ow)

    def run(self, src_ptr, dst_ptr):
        check(lib().amrb_prog_run(self.handle, C.c_void_p(src_ptr), C.c_void_p(dst_ptr), None, None, None,
                                  stream_ptr()))

    def __del__(self):
        h = getattr(self, "handle", None)
        if h is not None:
            try:
                lib().amrb_prog_destroy(h)
            except Exception:
                pass


def _packer(fa, to_staging, compact=False):
    key = ("plot_pack" if to_staging else "plot_unpack", compact)
    p = fa._native.get(key)
    if p is None:
        p = _Packer(fa, to_staging, compact)
        fa._native[key] = p
    return p


_pinned_lock = threading.Lock()
_pinned_free = {}  # element count -> [pinned float64 tensors]


def _pinned(n):
    with _pinned_lock:
        lst = _pinned_free.get(n)
        if lst:
            return lst.pop()
    return torch.empty(n, dtype=torch.float64, pin_memory=True)


def _pinned_release(t):
    with _pinned_lock:
        _pinned_free.setdefault(t.numel(), []).append(t)


class _LevelSnapshot:
    """A level packed on the device (caller's stream) and its copy-out to a
    pooled pinned buffer already enqueued (side stream): the writer thread only
    waits for the copy and writes."""

    def __init__(self, mesh):
        mesh.require_cuda("write_plotfile")
        p = _packer(mesh, True)
        self.p = p
        self.owners = [int(mesh.dm[i]) for i in range(len(mesh.ba))]
        self.nranks = mesh.dm.nranks
        self.dist = world_size() > 1
        self.rank = mesh.rank if self.dist else 0
        n = max(p.total // 8, 1)
        staging = torch.empty(n, dtype=torch.float64, device=mesh.device)
        main = torch.cuda.current_stream(mesh.device)
        p.run(mesh.storage.data_ptr(), staging.data_ptr())
        self.host = _pinned(n)
        side = torch.cuda.Stream(mesh.device)
        side.wait_stream(main)
        with torch.cuda.stream(side):
            self.host.copy_(staging, non_blocking=True)
        staging.record_stream(side)  # keep the block until the copy has read it
        self.copied = torch.cuda.Event()
        self.copied.record(side)

    def to_host(self):
        """Pinned host image of data.bin (records of boxes resident here)."""
        self.copied.synchronize()
        return self.host.numpy().view(np.uint8)

    def release(self):
        if self.host is not None:
            _pinned_release(self.host)
            self.host = None


def _write_level(fname, snap, image, nwriters, create):
    """Positioned writes of every record in waves of nwriters ranks
    (plotfile.py:195-241: same waves, same counters)."""
    p = snap.p
    if create:
        fd = os.open(fname, os.O_CREAT | os.O_WRONLY | os.O_TRUNC)
        if p.total:
            os.pwrite(fd, b"\0", p.total - 1)  # size the file up front
        os.close(fd)
    fd = os.open(fname, os.O_WRONLY)
    try:
        active = [0]
        gauge = threading.Lock()
        ranks = [snap.rank] if snap.dist else list(range(snap.nranks))

        def write_rank(rank, barrier):
            barrier.wait()  # the whole wave is live before anyone writes
            with gauge:
                active[0] += 1
                counters.peak("io_peak_writers", active[0])
            try:
                for i, r in enumerate(snap.owners):
                    if r != rank or not p.mine[i]:
                        continue
                    o, n = p.offsets[i], p.sizes[i]
                    os.pwrite(fd, memoryview(image[o : o + n]), o)
                    counters.incr("io_bytes_written", n)
            finally:
                with gauge:
                    active[0] -= 1

        for w0 in range(0, len(ranks), nwriters):
            wave = ranks[w0 : w0 + nwriters]
            counters.incr("io_waves")
            barrier = threading.Barrier(len(wave))
            threads = [threading.Thread(target=write_rank, args=(r, barrier)) for r in wave]
            for t in threads:
                t.start()
            for t in threads:
                t.join()
    finally:
        os.close(fd)


def _dist_barrier():
    if world_size() > 1:
        import torch.distributed as dist

        dist.barrier()


def _write_now(path, header_text, snaps, nwriters):
    root = not snaps or not snaps[0].dist or snaps[0].rank == 0
    if root:
        os.makedirs(path, exist_ok=True)
        with open(os.path.join(path, "Header"), "w") as fh:
            fh.write(header_text)
        for lev, s in enumerate(snaps):
            d = os.path.join(path, f"Level_{lev}")
            os.makedirs(d, exist_ok=True)
            fd = os.open(os.path.join(d, "data.bin"), os.O_CREAT | os.O_WRONLY | os.O_TRUNC)
            if s.p.total:
                os.pwrite(fd, b"\0", s.p.total - 1)
            os.close(fd)
    images = [s.to_host() for s in snaps]
    if snaps and snaps[0].dist:
        _dist_barrier()  # files exist and are sized before any rank writes
    try:
        for lev, (s, img) in enumerate(zip(snaps, images)):
            _write_level(os.path.join(path, f"Level_{lev}", "data.bin"), s, img, nwriters, create=False)
    finally:
        for s in snaps:
            s.release()


def write_plotfile(path, meshes, header, mode=None, transport=None):
    """Write one plotfile of device FabArrays; returns a WriteHandle (already
    done in static mode).  Bytes equal amrkit's write_plotfile (plotfile.py:244)."""
    if mode is None:
        mode = OutputMode.static(1)
    if len(meshes) != header.nlevels:
        raise ValueError("one mesh FabArray per header level required")
    text = _header_text(header, meshes)
    snaps = [_LevelSnapshot(m) for m in meshes]  # device pack, ordered before later kernels
    if mode.kind == "async":
        if snaps and snaps[0].dist:
            raise ValueError("asynchronous plotfiles need one process (the writer thread cannot join the "
                             "cross-rank barrier); use OutputMode.static under torchrun")
        return _writer.submit(lambda: _write_now(path, text, snaps, 1))
    _write_now(path, text, snaps, mode.nwriters)
    if snaps and snaps[0].dist:
        _dist_barrier()
    h = WriteHandle()
    h._finish()
    return h


class _Lines:
    def __init__(self, path):
        try:
            with open(path) as fh:
                self.lines = [ln.rstrip("\n") for ln in fh]
        except OSError as exc:
            raise IOError(f"cannot read header at {path}: {exc}") from exc
        self.at = 0

    def next(self, expect=None):
        line = self.lines[self.at]
        self.at += 1
        if expect is not None and not line.startswith(expect):
            raise ValueError(f"malformed header: wanted {expect!r}, got {line!r}")
        return line.split()


def _box(parts, dim):
    return Box(IntVect(int(x) for x in parts[:dim]), IntVect(int(x) for x in parts[dim : 2 * dim]))


def read_plotfile(path, nranks=1, device=None):
    """(header, meshes): metadata plus one ngrow=0 device FabArray per level
    (plotfile.py:314-360).  The records are copied to the device once per level
    and scattered into the FabArray by one copy-program launch."""
    rd = _Lines(os.path.join(path, "Header"))
    if rd.lines[0] != PLOTFILE_TAG:
        raise ValueError(f"not a plotfile (version tag {rd.lines[0]!r})")
    rd.at = 1
    rd.next("endian")
    rd.next("real")
    time = float(rd.next("time")[1])
    dim = int(rd.next("dim")[1])
    nlevels = int(rd.next("nlevels")[1])
    cp = rd.next("components")
    names = cp[2 : 2 + int(cp[1])]
    prob_lo = [float(x) for x in rd.next("prob_lo")[1:]]
    prob_hi = [float(x) for x in rd.next("prob_hi")[1:]]
    periodic = [bool(int(x)) for x in rd.next("periodic")[1:]]
    geoms, meshes = [], []
    for lev in range(nlevels):
        rd.next("level")
        dom = _box(rd.next("domain")[1:], dim)
        rd.next("cell_size")
        nboxes = int(rd.next("nboxes")[1])
        boxes, offs, sizes = [], [], []
        for _ in range(nboxes):
            parts = rd.next("box")[1:]
            boxes.append(_box(parts, dim))
            offs.append(int(parts[2 * dim]))
            sizes.append(int(parts[2 * dim + 1]))
        geoms.append(Geometry(dom, prob_lo, prob_hi, periodic))
        ba = BoxArray(boxes)
        dm = (DistributionMapping.single_rank(len(ba)) if nranks == 1
              else DistributionMapping([i % nranks for i in range(len(ba))], nranks))
        mesh = FabArray(ba, dm, ncomp=len(names), ngrow=0, device=device)
        p = _packer(mesh, False)
        if p.offsets != offs or p.sizes != sizes:
            raise ValueError(f"record table of level {lev} does not match the box layout")
        with open(os.path.join(path, f"Level_{lev}", "data.bin"), "rb") as fh:
            raw = np.frombuffer(fh.read(), dtype="<f8")
        if raw.nbytes != p.total:
            raise ValueError(f"data.bin of level {lev} has {raw.nbytes} bytes, header says {p.total}")
        staging = torch.from_numpy(raw.copy()).to(mesh.device) if raw.size else torch.zeros(1, dtype=torch.float64,
                                                                                          device=mesh.device)
        p.run(staging.data_ptr(), mesh.storage.data_ptr())
        torch.cuda.current_stream(mesh.device).synchronize()
        meshes.append(mesh)
    return PlotfileHeader(time, names, geoms), meshes


# ---------------------------------------------------------------------------
# checkpoints (mesh part; plotfile.py:466-524)
# ---------------------------------------------------------------------------


def write_checkpoint(path, meshes, header, step, user_blob=b"", pc=None, mode=None, transport=None):
    """Hierarchy metadata + level data + opaque payload (plotfile.py:466-488).
    Particle containers are outside this package's hot path."""
    if pc is not None:
        raise ValueError("particle checkpoints are not supported by the device writer (out of scope)")
    root = world_size() <= 1 or meshes[0].rank == 0
    if root:
        os.makedirs(path, exist_ok=True)
        lines = [CHECKPOINT_TAG, f"step {int(step)}", f"time {header.time!r}", f"nranks {meshes[0].dm.nranks}",
                 f"nlevels {len(meshes)}"]
        lines += [f"owners {lev} " + _ints(m.dm.owner) for lev, m in enumerate(meshes)]
        lines += [f"blob {len(user_blob)}", "particles 0"]
        with open(os.path.join(path, "Header"), "w") as fh:
            fh.write("\n".join(lines) + "\n")
        with open(os.path.join(path, "blob.bin"), "wb") as fh:
            fh.write(user_blob)
    write_plotfile(os.path.join(path, "mesh"), meshes, header, mode, transport).wait()


def read_checkpoint(path, device=None):
    """{step, time, nranks, owners, header, meshes, blob, particles} (plotfile.py:491-524)."""
    rd = _Lines(os.path.join(path, "Header"))
    if rd.lines[0] != CHECKPOINT_TAG:
        raise ValueError(f"not a checkpoint (version tag {rd.lines[0]!r})")
    rd.at = 1
    step = int(rd.next("step")[1])
    time = float(rd.next("time")[1])
    nranks = int(rd.next("nranks")[1])
    nlevels = int(rd.next("nlevels")[1])
    owners = [[int(x) for x in rd.next("owners")[2:]] for _ in range(nlevels)]
    nblob = int(rd.next("blob")[1])
    has_pc = bool(int(rd.next("particles")[1]))
    if has_pc:
        raise ValueError("checkpoint holds particles (not supported by the device reader)")
    with open(os.path.join(path, "blob.bin"), "rb") as fh:
        blob = fh.read()
    if len(blob) != nblob:
        raise ValueError("checkpoint blob length mismatch")
    header, meshes = read_plotfile(os.path.join(path, "mesh"), device=device)
    return {"step": step, "time": time, "nranks": nranks, "owners": owners, "header": header, "meshes": meshes,
            "blob": blob, "particles": None}
