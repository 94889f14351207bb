import torch, numpy as np
n = 256**3 * 2  # 268 MB of fp64
a = torch.randn(n, dtype=torch.float64, device="cuda"); b = torch.randn(n, dtype=torch.float64, device="cuda")
c = torch.empty_like(a)
def t(fn, reps=20):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e-3
ts = t(lambda: torch.sum(a)); print(f"sum(a) read-only {8*n/ts/1e9:.0f} GB/s")
ts = t(lambda: torch.amax(a)); print(f"amax(a) read-only {8*n/ts/1e9:.0f} GB/s")
ts = t(lambda: torch.linalg.vector_norm(a - b, float('inf'))); print(f"inf-norm(a-b) (2 kernels, temp) {8*n*4/ts/1e9:.0f} GB/s effective incl. temp")
ts = t(lambda: torch.add(a, b, out=c)); print(f"c = a + b (2R 1W) {24*n/ts/1e9:.0f} GB/s")
ts = t(lambda: c.copy_(a)); print(f"copy {16*n/ts/1e9:.0f} GB/s")
h = n // 2
ts = t(lambda: torch.add(a[:h], b[:h], out=c[:h])); print(f"half-size add {24*h/ts/1e9:.0f} GB/s")
