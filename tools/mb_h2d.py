"""Host<->device copy bandwidth with every rank copying at once (the e2e leg
of bench.py at N GPUs), with and without binding each rank's CPU affinity
(hence its pinned pages, first touch) to its GPU's NUMA node.

torchrun --nproc-per-node N tools/mb_h2d.py [bind]"""
import os
import sys
import time

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2009_12009_b200.hostaffinity import bind_to_gpu  # noqa: E402

rank = int(os.environ.get("RANK", 0))
world = int(os.environ.get("WORLD_SIZE", 1))
torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", 0)))
dist.init_process_group("gloo" if world == 1 else "nccl", init_method="env://")
bind = len(sys.argv) > 1 and sys.argv[1] == "bind"
cpus = bind_to_gpu(torch.cuda.current_device()) if bind else None
n = 256 ** 3
h_in = torch.empty(n, dtype=torch.float64).pin_memory()
h_out = torch.empty(n, dtype=torch.float64).pin_memory()
h_in.fill_(1.0)
d = torch.empty(n, dtype=torch.float64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
for mode in ("h2d", "d2h", "both"):
    for it in range(4):
        dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        if mode in ("h2d", "both"):
            with torch.cuda.stream(s1):
                d.copy_(h_in, non_blocking=True)
        if mode in ("d2h", "both"):
            with torch.cuda.stream(s2):
                h_out.copy_(d, non_blocking=True)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
    nb = 8 * n * (2 if mode == "both" else 1)
    t = torch.tensor([dt], device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    if rank == 0:
        print(f"world={world} bind={bind} {mode:5s} per-rank {nb / dt / 1e9:6.1f} GB/s  "
              f"aggregate {world * nb / t.item() / 1e9:6.1f} GB/s  (rank0 cpus {None if cpus is None else len(cpus)})",
              flush=True)
dist.destroy_process_group()
