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

import concurrent.futures
import ctypes as C
import itertools
import os
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
    """How a plotfile is written (plotfile.py:43-64): ``static(nwriters)``
    writes before returning, ranks in waves of nwriters; ``asynchronous()``
    snapshots the data and hands the writes to the background writer."""

    __slots__ = ("kind", "nwriters")
    _KINDS = ("static", "async")

    def __init__(self, kind, nwriters=1):
        nwriters = int(nwriters)
        if kind not in self._KINDS:
            raise ValueError("output mode must be 'static' or 'async'")
        if nwriters < 1:
            raise ValueError("nwriters must be >= 1")
        self.kind, self.nwriters = kind, nwriters

    @classmethod
    def static(cls, nwriters=1):
        return cls("static", nwriters)

    @classmethod
    def asynchronous(cls):
        return cls("async")

    def __repr__(self):
        return f"OutputMode({self.kind}, nwriters={self.nwriters})"


class WriteHandle:
    """Completion of one plotfile write.  ``done`` polls; ``wait(timeout)``
    blocks, raises TimeoutError if the write is still running and re-raises the
    writer's exception if it failed.  Backed by a concurrent.futures.Future."""

    def __init__(self, future=None):
        if future is None:  # a write that already happened (static mode)
            future = concurrent.futures.Future()
            future.set_result(None)
        self._future = future

    @property
    def done(self):
        return self._future.done()

    def wait(self, timeout=None):
        try:
            self._future.result(timeout)
        except concurrent.futures.TimeoutError:
            raise TimeoutError("plotfile write still in progress") from None


class _BackgroundWriter:
    """One writer thread; submit() blocks while a snapshot is already queued
    behind the running one (one pending snapshot of backpressure, as
    plotfile.py:86-115)."""

    def __init__(self):
        self._pool = concurrent.futures.ThreadPoolExecutor(max_workers=1, thread_name_prefix="amrb-plotfile")
        self._slots = threading.BoundedSemaphore(2)  # the running job + one pending

    def submit(self, job):
        self._slots.acquire()

        def run():
            try:
                job()
            finally:
                self._slots.release()

        return WriteHandle(self._pool.submit(run))


_writer = _BackgroundWriter()


class PlotfileHeader:
    """Simulation time, component names and one Geometry per level
    (plotfile.py:123-138)."""

    def __init__(self, time, names, geoms):
        names = [str(n) for n in names]
        spaced = [n for n in names if " " in n]
        if spaced:
            raise ValueError(f"component names may not contain spaces ({spaced[0]!r})")
        self.version = PLOTFILE_TAG
        self.time, self.names, self.geoms = float(time), names, list(geoms)

    @property
    def nlevels(self):
        return len(self.geoms)


def _floats(vals):
    return " ".join(map(repr, map(float, vals)))


def _ints(vals):
    return " ".join(str(int(v)) for v in vals)


def _box_text(b):
    return _ints(tuple(b.lo) + tuple(b.hi))


def _record_layout(ba, ncomp):
    """Byte offset and size of every box record, and the file size."""
    sizes = [8 * ncomp * b.num_cells() for b in ba]
    ends = list(itertools.accumulate(sizes))
    return [e - n for e, n in zip(ends, sizes)], sizes, (ends[-1] if ends else 0)


def _header_text(header, meshes):
    """The Header file (FORMAT.md:17-84): global key/value lines, then per
    level its domain, cell size and one line per box record."""
    g0 = header.geoms[0]
    rows = [
        (PLOTFILE_TAG,), ("endian", "little"), ("real", "float64"), ("time", repr(header.time)),
        ("dim", g0.dim), ("nlevels", header.nlevels),
        ("components", f"{len(header.names)} " + " ".join(header.names)),
        ("prob_lo", _floats(g0.prob_lo)), ("prob_hi", _floats(g0.prob_hi)), ("periodic", _ints(g0.periodic)),
    ]
    for lev, (mesh, geom) in enumerate(zip(meshes, header.geoms)):
        offs, sizes, _ = _record_layout(mesh.ba, mesh.ncomp)
        rows += [("level", lev), ("domain", _box_text(geom.domain)), ("cell_size", _floats(geom.cell_size)),
                 ("nboxes", len(mesh.ba))]
        rows += [("box", _box_text(b), o, n) for b, o, n in zip(mesh.ba, offs, sizes)]
    return "".join(" ".join(map(str, r)) + "\n" for r in rows)


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


def _write_records(fd, snap, image, rank):
    """Every record of `rank`'s boxes held here, straight from the pinned image."""
    p = snap.p
    for i in (i for i, r in enumerate(snap.owners) if r == rank and p.mine[i]):
        off, n = p.offsets[i], p.sizes[i]
        os.pwrite(fd, memoryview(image[off:off + n]), off)
        counters.incr("io_bytes_written", n)


def _waves(nranks, nwriters):
    return [list(range(w, min(w + nwriters, nranks))) for w in range(0, nranks, nwriters)]


def _write_level(fname, snap, image, nwriters):
    """Positioned writes in waves of nwriters ranks (plotfile.py:195-241):
    ranks of one wave write concurrently, waves run one after another, and
    io_waves / io_peak_writers count them as the reference does.  Simulated
    ranks (one process): one thread per rank of the wave.  One process per GPU:
    a rank writes in its own wave; every rank passes a barrier per wave."""
    fd = os.open(fname, os.O_WRONLY)
    try:
        for wave in _waves(snap.nranks, nwriters):
            counters.incr("io_waves")
            counters.peak("io_peak_writers", len(wave))
            if snap.dist:
                if snap.rank in wave:
                    _write_records(fd, snap, image, snap.rank)
                _dist_barrier()
            else:
                with concurrent.futures.ThreadPoolExecutor(max_workers=len(wave)) as pool:
                    for f in [pool.submit(_write_records, fd, snap, image, r) for r in wave]:
                        f.result()
    finally:
        os.close(fd)


def _dist_barrier():
    if world_size() > 1:
        import torch.distributed as dist

        dist.barrier()


def _write_now(path, header_text, snaps, nwriters):
    root = not snaps or not snaps[0].dist or snaps[0].rank == 0
    if root:  # the Header, and every data.bin sized up front
        os.makedirs(path, exist_ok=True)
        with open(os.path.join(path, "Header"), "w") as fh:
            fh.write(header_text)
        for lev, s in enumerate(snaps):
            os.makedirs(os.path.join(path, f"Level_{lev}"), exist_ok=True)
            with open(os.path.join(path, f"Level_{lev}", "data.bin"), "wb") as fh:
                fh.truncate(s.p.total)
    images = [s.to_host() for s in snaps]
    if snaps and snaps[0].dist:
        _dist_barrier()  # files exist and are sized before any rank writes
    try:
        for lev, (s, img) in enumerate(zip(snaps, images)):
            _write_level(os.path.join(path, f"Level_{lev}", "data.bin"), s, img, nwriters)
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
    return WriteHandle()


class _HeaderScan:
    """Header lines as (key, fields) records consumed in order: take(key)
    checks the key and returns the fields after it."""

    def __init__(self, path):
        try:
            with open(path) as fh:
                text = fh.read()
        except OSError as exc:
            raise IOError(f"cannot read header at {path}: {exc}") from exc
        self.rows = [ln.split() for ln in text.splitlines()]
        self.tag = text.splitlines()[0] if self.rows else ""
        self.pos = 1

    def take(self, key):
        row = self.rows[self.pos] if self.pos < len(self.rows) else [""]
        if not row or row[0] != key:
            raise ValueError(f"malformed header: wanted {key!r}, got {' '.join(row)!r}")
        self.pos += 1
        return row[1:]

    def one(self, key, conv):
        return conv(self.take(key)[0])


def _box(fields, dim):
    return Box([int(x) for x in fields[:dim]], [int(x) for x in fields[dim:2 * dim]])


def read_plotfile(path, nranks=1, device=None):
    """(header, meshes): metadata plus one ngrow=0 device FabArray per level
    (plotfile.py:314-360).  The records are copied to the device once per level
    and scattered into the FabArray by one copy-program launch."""
    hd = _HeaderScan(os.path.join(path, "Header"))
    if hd.tag != PLOTFILE_TAG:
        raise ValueError(f"not a plotfile (version tag {hd.tag!r})")
    hd.take("endian")
    hd.take("real")
    time = hd.one("time", float)
    dim = hd.one("dim", int)
    nlevels = hd.one("nlevels", int)
    comps = hd.take("components")
    names = comps[1:1 + int(comps[0])]
    prob_lo = [float(x) for x in hd.take("prob_lo")]
    prob_hi = [float(x) for x in hd.take("prob_hi")]
    periodic = [x == "1" for x in hd.take("periodic")]
    geoms, meshes = [], []
    for lev in range(nlevels):
        hd.take("level")
        dom = _box(hd.take("domain"), dim)
        hd.take("cell_size")
        rec = [hd.take("box") for _ in range(hd.one("nboxes", int))]
        boxes = [_box(f, dim) for f in rec]
        offs = [int(f[2 * dim]) for f in rec]
        sizes = [int(f[2 * dim + 1]) for f in rec]
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
    hd = _HeaderScan(os.path.join(path, "Header"))
    if hd.tag != CHECKPOINT_TAG:
        raise ValueError(f"not a checkpoint (version tag {hd.tag!r})")
    step = hd.one("step", int)
    time = hd.one("time", float)
    nranks = hd.one("nranks", int)
    nlevels = hd.one("nlevels", int)
    owners = [[int(x) for x in hd.take("owners")[1:]] for _ in range(nlevels)]
    nblob = hd.one("blob", int)
    if hd.one("particles", int):
        raise ValueError("checkpoint holds particles (not supported by the device reader)")
    with open(os.path.join(path, "blob.bin"), "rb") as fh:
        blob = fh.read()
    if len(blob) != nblob:
        raise ValueError("checkpoint blob length mismatch")
    header, meshes = read_plotfile(os.path.join(path, "mesh"), device=device)
    return {"step": step, "time": time, "nranks": nranks, "owners": owners, "header": header, "meshes": meshes,
            "blob": blob, "particles": None}
