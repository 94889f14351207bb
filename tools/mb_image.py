import sys, time, torch, numpy as np
sys.path.insert(0, '/root/repo')
import paper_2009_12009_b200 as A
from paper_2009_12009_b200.plotfile import _packer
dom = A.Box((0,0,0),(255,255,255)); ba = A.BoxArray([dom]).max_size(64)
dm = A.DistributionMapping.single_rank(len(ba))
fa = A.MultiFab(ba, dm, 1, 0); fa.storage.normal_()
img = torch.empty(fa.image_size(), dtype=torch.float64).pin_memory()
dev = torch.empty(fa.image_size(), dtype=torch.float64, device="cuda")
def wall(fn, n=5):
    fn(); torch.cuda.synchronize(); ts = []
    for _ in range(n):
        t0 = time.perf_counter(); fn(); torch.cuda.synchronize(); ts.append(time.perf_counter() - t0)
    return min(ts) * 1e3
print("H2D 134MB pinned->dev contiguous: %.2f ms" % wall(lambda: dev.copy_(img, non_blocking=True)))
print("D2H dev->pinned contiguous:       %.2f ms" % wall(lambda: img.copy_(dev, non_blocking=True)))
print("from_host_image:                  %.2f ms" % wall(lambda: fa.from_host_image(img)))
print("to_host_image:                    %.2f ms" % wall(lambda: fa.to_host_image(img)))
up = _packer(fa, False, compact=True); dn = _packer(fa, True, compact=True)
print("scatter launch:                   %.3f ms" % wall(lambda: up.run(dev.data_ptr(), fa.storage.data_ptr())))
print("gather launch:                    %.3f ms" % wall(lambda: dn.run(fa.storage.data_ptr(), dev.data_ptr())))
host = {i: f.valid().detach().cpu().pin_memory() for i, f in fa.fabs.items()}
def perbox():
    for i, t in host.items(): fa.fab(i).valid().copy_(t, non_blocking=True)
print("per-box H2D (64 copies):          %.2f ms" % wall(perbox))
