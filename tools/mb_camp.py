"""Partition-camping probe: residual-norm kernel on (phi, rhs) with rhs's
storage re-based by various byte offsets (same layout, same values)."""
import ctypes as C, sys, numpy as np, torch
sys.path.insert(0, '/root/repo')
import paper_2009_12009_b200 as A
from paper_2009_12009_b200._native import lib, check
from paper_2009_12009_b200.device import level_of, field_of, stream_ptr, dh_array
dom = A.Box((0,0,0),(255,255,255)); ba = A.BoxArray([dom])
dm = A.DistributionMapping.single_rank(1)
phi = A.MultiFab(ba, dm, 1, 1); phi.storage.normal_()
rhs = A.MultiFab(ba, dm, 1, 0)
n = rhs.storage.numel()
big = torch.empty(n + (1 << 20), dtype=torch.float64, device="cuda")
out = torch.zeros(1, dtype=torch.float64, device="cuda")
dh = dh_array((65536.0,) * 3)
def run():
    check(lib().amrb_residual_norm(level_of(phi).handle, field_of(rhs).handle, C.c_void_p(rhs.storage.data_ptr()),
                                   field_of(phi).handle, C.c_void_p(phi.storage.data_ptr()), dh,
                                   C.c_void_p(out.data_ptr()), stream_ptr()))
for off_b in (0, 256, 512, 1024, 2048, 4096, 8192, 65536, 1 << 20, (1 << 20) + 4096):
    rhs.storage = big[off_b // 8 : off_b // 8 + n]
    rhs.storage.normal_()
    run(); torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph(); s = torch.cuda.Stream(); s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            for _ in range(20): run()
    torch.cuda.synchronize(); ts = []
    for _ in range(5):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); g.replay(); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1) * 1e3 / 20)
    d = (rhs.storage.data_ptr() - phi.storage.data_ptr()) % (1 << 21)
    print(f"rhs offset {off_b:8d} B (base delta mod 2MiB {d:8d}): resid_norm {np.median(ts):6.1f} us")
