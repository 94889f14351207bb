"""Pin a rank's host threads to the CPUs next to its GPU.

The end-to-end path (bench.py ``e2e``; the FabArray host images) streams every
step's rhs in and solution out through pinned host buffers.  With N ranks
copying at once the host side is the shared resource: a rank whose threads --
and so, by first touch, whose pinned pages -- sit on the far socket sends its
copies across the CPU interconnect.  ``bind_to_gpu`` restricts the calling
process to the CPUs NVML reports as local to the GPU (intersected with the
CPUs the process may use), before the pinned buffers are allocated.
"""

from __future__ import annotations

import os

__all__ = ["bind_to_gpu", "gpu_local_cpus"]


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
