import torch
n = 256**3
x = torch.randn(2*n, dtype=torch.float64, device='cuda'); y = torch.empty_like(x)
a = torch.randn(n, dtype=torch.float64, device='cuda'); b = torch.randn(n, dtype=torch.float64, device='cuda'); c = torch.empty_like(a)
for name, fn, nbytes in (("copy 268MB", lambda: y.copy_(x), 2*2*n*8), ("a+b->c (3x134MB)", lambda: torch.add(a, b, out=c), 3*n*8)):
    for _ in range(3): fn()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20): fn()
    e1.record(); torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / 20 * 1e3
    print(f"{name}: {t:.1f} us  {nbytes/t/1e3:.0f} GB/s")
