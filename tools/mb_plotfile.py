"""C3-size plotfile write (256^3, 64 boxes of 64^3, 1 comp = 134 MB): device
pack + copy-out + pwrite, async overlap with MLMG cycles, and the reference's
host algorithm (per-box contiguous copy + tobytes + pwrite) on host arrays."""
import os, sys, time, shutil, numpy as np, torch
sys.path.insert(0, '/root/repo')
import paper_2009_12009_b200 as A
from paper_2009_12009_b200.plotfile import _LevelSnapshot
out = os.environ.get("PLT_DIR", "/tmp/amrb_plt")
dom = A.Box((0,0,0),(255,255,255)); ba = A.BoxArray([dom]).max_size(64)
dm = A.DistributionMapping.single_rank(len(ba))
fa = A.MultiFab(ba, dm, 1, 1); fa.storage.normal_()
geom = A.Geometry(dom, (0.0,)*3, (1.0,)*3, True)
hdr = A.PlotfileHeader(0.5, ["phi"], [geom])
def t_sync():
    shutil.rmtree(out, ignore_errors=True); torch.cuda.synchronize(); t0 = time.perf_counter()
    A.write_plotfile(out, [fa], hdr).wait(); return time.perf_counter() - t0
for _ in range(2): t_sync()
ts = [t_sync() for _ in range(3)]
nb = 8 * ba.num_cells()
print(f"static write 134 MB: {min(ts)*1e3:.1f} ms  ({nb/min(ts)/1e9:.2f} GB/s end to end)")
# pieces: device pack, copy-out
torch.cuda.synchronize()
e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
from paper_2009_12009_b200.plotfile import _packer
p = _packer(fa, True); stg = torch.empty(nb // 8, dtype=torch.float64, device="cuda")
for _ in range(3): p.run(fa.storage.data_ptr(), stg.data_ptr())
torch.cuda.synchronize(); e0.record()
for _ in range(10): p.run(fa.storage.data_ptr(), stg.data_ptr())
e1.record(); torch.cuda.synchronize(); tp = e0.elapsed_time(e1) / 10
print(f"  device pack (1 launch): {tp*1e3:.1f} us  ({2*nb/tp/1e6:.0f} GB/s r+w)")
t0 = time.perf_counter(); s = _LevelSnapshot(fa); img = s.to_host(); t1 = time.perf_counter(); s.release()
print(f"  snapshot (pack + copy-out to pinned): {(t1-t0)*1e3:.1f} ms ({nb/(t1-t0)/1e9:.1f} GB/s)")
# async overlap: submit, then run V-cycles; compare cycle time with/without a concurrent write
mg = A.MLMG(geom, ba, dm, transport=A.Transport(1))
rhs = A.MultiFab(ba, dm, 1, 0)
for f in rhs.fabs.values(): f.valid().normal_()
mu = sum(float(f.valid().sum()) for f in rhs.fabs.values()) / ba.num_cells()
for f in rhs.fabs.values(): f.valid().sub_(mu)
phi = A.MultiFab(ba, dm, 1, 1)
mg.solve(phi, rhs, rtol=1e-10, max_iter=3)
def solve_time():
    torch.cuda.synchronize(); t0 = time.perf_counter(); phi.setval(0.0); mg.solve(phi, rhs, rtol=1e-10, max_iter=100)
    torch.cuda.synchronize(); return time.perf_counter() - t0
base = min(solve_time() for _ in range(3))
shutil.rmtree(out, ignore_errors=True)
t0 = time.perf_counter(); h = A.write_plotfile(out, [fa], hdr, A.OutputMode.asynchronous()); t_sub = time.perf_counter() - t0
ov = solve_time(); h.wait(); t_all = time.perf_counter() - t0
print(f"async: submit returns in {t_sub*1e3:.2f} ms; solve alone {base*1e3:.2f} ms, solve during the write {ov*1e3:.2f} ms; write done after {t_all*1e3:.1f} ms")
# reference algorithm on host arrays (what amrkit does per box)
host = [fa.fab(i).valid().cpu().numpy() for i in range(len(ba))]
def t_ref():
    shutil.rmtree(out + "_ref", ignore_errors=True); os.makedirs(out + "_ref/Level_0")
    t0 = time.perf_counter()
    fn = out + "_ref/Level_0/data.bin"; fd = os.open(fn, os.O_CREAT | os.O_WRONLY | os.O_TRUNC)
    os.pwrite(fd, b"\0", nb - 1); off = 0
    for a in host:
        d = np.ascontiguousarray(a).astype("<f8", copy=False).tobytes(); os.pwrite(fd, d, off); off += len(d)
    os.close(fd); return time.perf_counter() - t0
tr = min(t_ref() for _ in range(3))
print(f"reference host algorithm (data already on host): {tr*1e3:.1f} ms ({nb/tr/1e9:.2f} GB/s)")
same = open(out + "_ref/Level_0/data.bin", "rb").read() == open(out + "/Level_0/data.bin", "rb").read()
print("data.bin identical to the host-algorithm bytes:", same)
