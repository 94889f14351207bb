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

# ---- CPU binding to the GPU's NUMA-local CPUs (NVML) ----------------------------
def _nvml_handle(pynvml, device_index):
    import torch

    props = torch.cuda.get_device_properties(device_index)
    bus = getattr(props, "pci_bus_id", None)
    dom = getattr(props, "pci_domain_id", 0)
    dev = getattr(props, "pci_device_id", 0)
    if bus is not None:
        pci = f"{dom:08x}:{bus:02x}:{dev:02x}.0".encode()
        try:
            return pynvml.nvmlDeviceGetHandleByPciBusId(pci)
        except pynvml.NVMLError:
            pass
    # no PCI identity from torch: CUDA ordinal == NVML ordinal unless remapped
    vis = os.environ.get("CUDA_VISIBLE_DEVICES")
    idx = device_index
    if vis:
        ids = [v.strip() for v in vis.split(",") if v.strip()]
        if device_index < len(ids) and ids[device_index].isdigit():
            idx = int(ids[device_index])
    return pynvml.nvmlDeviceGetHandleByIndex(idx)


def gpu_local_cpus(device_index):
    """The set of CPU ids NVML reports as close to CUDA device ``device_index``
    (None if NVML is unavailable)."""
    try:
        import pynvml
    except ImportError:
        return None
    try:
        pynvml.nvmlInit()
    except Exception:
        return None
    try:
        h = _nvml_handle(pynvml, device_index)
        ncpu = os.cpu_count() or 1
        words = (ncpu + 63) // 64
        mask = pynvml.nvmlDeviceGetCpuAffinity(h, words)
        cpus = set()
        for w, m in enumerate(mask):
            m = int(m)
            for b in range(64):
                if (m >> b) & 1:
                    cpus.add(64 * w + b)
        return cpus or None
    except Exception:
        return None
    finally:
        try:
            pynvml.nvmlShutdown()
        except Exception:
            pass


def bind_to_gpu(device_index):
    """Restrict this process to the CPUs local to ``device_index``; returns the
    CPU set applied, or None (nothing changed: no NVML, or no overlap with the
    CPUs this process may use)."""
    cpus = gpu_local_cpus(device_index)
    if not cpus:
        return None
    allowed = os.sched_getaffinity(0)
    use = cpus & allowed
    if not use or use == allowed:
        return None if not use else use
    os.sched_setaffinity(0, use)
    return use


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
